# round 2, call B: class-split initial pass -- correctness on scaled configs, then rmat24 probe
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2b
mkdir -p $OUT
( timeout 300 python tools/class_probe.py rmat24 1 0 ) > $OUT/probe_first.log 2>&1
( timeout 900 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
( timeout 600 python tools/class_probe.py rmat24 5 0 1 ) > $OUT/probe_rmat24.log 2>&1
for bps in 2; do ( GCOL_K1H_BPS=$bps PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_bps$bps.log 2>&1; done
( GCOL_K1H_DRIFT=0 PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_drift0.log 2>&1
( GCOL_K1H_RECHECK=0 PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_norecheck.log 2>&1
( GCOL_CLASS_T=32 PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_T32.log 2>&1
