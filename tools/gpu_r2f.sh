set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2f
mkdir -p $OUT
( timeout 900 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu2.log 2>&1
( PROBE_VERIFY=0 GCOL_K1_PROFILE=1 timeout 900 python tools/class_probe.py rmat27 2 0 1 ) > "$OUT/probeM_rmat27.log" 2>&1
( PROBE_VERIFY=0 GCOL_K1H_ROWW=3 timeout 900 python tools/class_probe.py rmat27 2 0 ) > "$OUT/probeM_rmat27_rw3.log" 2>&1
