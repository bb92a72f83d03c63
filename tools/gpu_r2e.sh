set -x
export PYTHONUNBUFFERED=1 GCOL_K1_PROFILE=1
OUT=gpurun_out/r2e
mkdir -p $OUT
( timeout 300 python tools/class_probe.py rmat24 3 0 ) > $OUT/probe_d2.log 2>&1
export PROBE_VERIFY=0
( GCOL_K1H_DRIFT=0 timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_d0.log 2>&1
( GCOL_K1H_DRIFT=4 timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_d4.log 2>&1
( GCOL_K1H_BPS=2 timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_b2.log 2>&1
( timeout 900 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
