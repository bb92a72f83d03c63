set -x
export PYTHONUNBUFFERED=1
timeout 120 python tools/one_run.py stencil > gpurun_out/one_stencil.log 2>&1; echo rc=$? >> gpurun_out/one_stencil.log
GCOL_TRACE=1 timeout 300 python tools/dbg_run.py --config stencil --steps 3 --warmup 3 > gpurun_out/dbg_stencil.json 2> gpurun_out/dbg_stencil.err; echo rc=$? >> gpurun_out/dbg_stencil.err
for c in tri er stencil; do
GCOL_EAGER=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -f -o gpurun_out/k1w_$c python tools/one_run.py $c > gpurun_out/ncu_$c.log 2>&1
done
