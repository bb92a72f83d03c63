set -x
export PYTHONUNBUFFERED=1 PROBE_VERIFY=0
OUT=gpurun_out/r2f
mkdir -p $OUT
( GCOL_K1H_COMPACT=1 PROBE_VERIFY=1 timeout 300 python tools/class_probe.py rmat24 2 0 ) > "$OUT/probeW_c24.log" 2>&1
( timeout 900 python tools/class_probe.py rmat27 2 0 ) > "$OUT/probeW_c27.log" 2>&1
( GCOL_K1H_COMPACT=0 timeout 900 python tools/class_probe.py rmat27 1 0 ) > "$OUT/probeW_nc27.log" 2>&1
( GCOL_K1H_COMPACT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "class_split or concurrent" ) > $OUT/pytest_cls3.log 2>&1
