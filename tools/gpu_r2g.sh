set -x
export PYTHONUNBUFFERED=1 PROBE_VERIFY=0 GCOL_EAGER=1
OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_heavy -c 1 -o $OUT/k1h python tools/class_probe.py rmat24 1 0 > $OUT/ncu_k1h.log 2>&1
