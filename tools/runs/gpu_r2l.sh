# round 2, call L: CLI tests on the GPU; K1H after removing the compact-mode branch (R-MAT 24 probe, R-MAT 27 bench)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2l
mkdir -p $OUT
( timeout 600 python -m pytest tests/test_gpu_cli.py -m gpu -x -q ) > $OUT/pytest_cli.log 2>&1; echo "rc=$?" >> $OUT/pytest_cli.log
tail -5 $OUT/pytest_cli.log
( GCOL_K1_PROFILE=1 PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_rmat24.log 2>&1
tail -3 $OUT/probe_rmat24.log | cut -c1-330
( timeout 1500 python bench.py --config rmat24 --steps 10 --warmup 3 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err; echo "rc=$?"
cut -c1-700 $OUT/bench_rmat24.json
( timeout 2400 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err; echo "rc=$?"
cut -c1-700 $OUT/bench_rmat27.json
