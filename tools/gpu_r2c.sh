# round 2, call C: K1H with hinted polling -- probes + ncu of both class passes
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2c
mkdir -p $OUT
( timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe.log 2>&1
for v in "GCOL_K1H_RECHECK=0" "GCOL_K1H_DRIFT=3" "GCOL_K1H_DRIFT=1" "GCOL_K1H_BPS=2 GCOL_K1H_DRIFT=1"; do
  ( env $v PROBE_VERIFY=0 timeout 300 python tools/class_probe.py rmat24 3 0 ) > "$OUT/probe_${v// /_}.log" 2>&1
done
export GCOL_EAGER=1 PROBE_VERIFY=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_heavy -c 1 -o $OUT/k1h python tools/class_probe.py rmat24 1 0 > $OUT/ncu_k1h.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -o $OUT/k1l python tools/class_probe.py rmat24 1 0 > $OUT/ncu_k1l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/class_probe.py rmat24 1 0 > $OUT/ncu_launches.log 2>&1
