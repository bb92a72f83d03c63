set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2f
mkdir -p $OUT
( timeout 900 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu3.log 2>&1
( timeout 900 python bench.py --config rmat24 --steps 5 --warmup 3 --no-cpu-baseline ) > $OUT/bench24_e2e.json 2> $OUT/bench24_e2e.err
( timeout 1200 python bench.py --config rmat27 --steps 5 --warmup 3 --no-cpu-baseline ) > $OUT/bench27_e2e.json 2> $OUT/bench27_e2e.err
