set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2f
mkdir -p $OUT
( timeout 1200 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu5.log 2>&1
