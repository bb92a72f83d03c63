# Round profiling pass (tooling): bench lines for the four single-GPU
# configs, the ncu launch list of the default bench command, one
# `ncu --set full` capture of K1 per config, and an R-MAT drift-bound sweep.
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/prof
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
for c in tri er stencil rmat24; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_tri.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > $OUT/launches_tri.log 2>&1
for c in tri er stencil; do
  GCOL_EAGER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -f \
    -o $OUT/k1_$c python tools/one_run.py $c > $OUT/ncu_$c.log 2>&1
done
GCOL_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_pipe -c 1 -f \
  -o $OUT/k1_rmat24 python tools/one_run.py rmat24 > $OUT/ncu_rmat24.log 2>&1
for d in 2 3 4 6 0; do
  GCOL_K1_DRIFT=$d timeout 600 python tools/k1_ab.py rmat24 --variants 0 --runs 5 | sed "s/^{/{\"drift\":$d,/"
done > $OUT/rmat_drift.jsonl 2> $OUT/rmat_drift.err
