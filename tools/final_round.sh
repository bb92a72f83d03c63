# End-of-round refresh (tooling): GPU tests, smoke, bench lines for the four
# single-GPU configs, ncu captures of K1W on ER (occupancy heuristic) and the
# eager launch list of the default bench command.
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/final
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
for c in tri er stencil rmat24; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_tri.json 2> $OUT/bench_reference_tri.err
GCOL_EAGER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -f \
  -o $OUT/k1_er python tools/one_run.py er > $OUT/ncu_er.log 2>&1
GCOL_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_tri_eager.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > $OUT/launches_tri.log 2>&1
