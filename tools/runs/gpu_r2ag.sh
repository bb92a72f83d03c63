# round 2, call AG: short-budget waiting heavy pass as the default for L2-resident skewed graphs: full GPU suite, R-MAT 24 + 27 bench
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ag
mkdir -p $OUT
( timeout 1800 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
( timeout 1500 python bench.py --config rmat24 --steps 10 --warmup 3 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err; echo "rc=$?"
cut -c1-300 $OUT/bench_rmat24.json
( timeout 2400 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err; echo "rc=$?"
cut -c1-300 $OUT/bench_rmat27.json
( timeout 600 python tools/compare_algorithms.py 2>&1 | tail -20 ) > $OUT/compare.log 2>&1
