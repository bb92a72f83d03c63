set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2f
mkdir -p $OUT
( timeout 600 python -m pytest tests/test_gpu_dist.py -x -q ) > $OUT/pytest_dist.log 2>&1
( timeout 1200 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu6.log 2>&1
( timeout 600 python bench.py --config rmat24 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --distributed ) > $OUT/bench_dist24.json 2> $OUT/bench_dist24.err
( timeout 600 python bench.py --gpus 2 --config tri --steps 3 --warmup 3 ) > $OUT/bench_gpus2.json 2> $OUT/bench_gpus2.err; echo "rc=$?" >> $OUT/bench_gpus2.err
