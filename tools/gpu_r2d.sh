set -x
export PYTHONUNBUFFERED=1 PROBE_VERIFY=0 GCOL_K1_PROFILE=1
OUT=gpurun_out/r2d
mkdir -p $OUT
( timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_d2.log 2>&1
( GCOL_K1H_DRIFT=0 timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_d0.log 2>&1
( GCOL_K1H_BPS=2 GCOL_K1H_DRIFT=0 timeout 300 python tools/class_probe.py rmat24 2 0 ) > $OUT/probe_b2d0.log 2>&1
