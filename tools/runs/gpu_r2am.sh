# round 2, call AM: final validation of the final tree: GPU suite, smoke, default bench (R-MAT 27), R-MAT 24 bench, launch list
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2am
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
( timeout 1800 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log; cat $OUT/smoke.log
( timeout 2400 python bench.py ) > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "rc=$?"
cut -c1-260 $OUT/bench_default.json
( timeout 1500 python bench.py --config rmat24 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err; echo "rc=$?"
cut -c1-260 $OUT/bench_rmat24.json
KRE='regex:k1_|k_mark|k_cand|k_list|k_heavy|k_control|k_verify|k_census|k_class|k_check|k_graph'
GCOL_EAGER=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_rmat27.log 2>&1
GCOL_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat24.csv python tools/one_run.py rmat24 > $OUT/launches_rmat24.log 2>&1
