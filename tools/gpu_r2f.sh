set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2f
mkdir -p $OUT
( timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "class_split or concurrent" ) > $OUT/pytest_class.log 2>&1
( timeout 1200 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu4.log 2>&1
