set -x
export PYTHONUNBUFFERED=1 PROBE_VERIFY=0
OUT=gpurun_out/r2f
mkdir -p $OUT
for v in "4 6" "4 8" "5 6" "5 8"; do set -- $v
( GCOL_K1H_ROWW=$1 GCOL_K1H_PIECEW=$2 timeout 900 python tools/class_probe.py rmat27 1 0 ) > "$OUT/probeS_rmat27_rw$1_pw$2.log" 2>&1
done
( GCOL_K1H_ROWW=4 GCOL_K1H_PIECEW=6 timeout 900 python tools/class_probe.py rmat24 2 0 ) > "$OUT/probeS_rmat24_rw4_pw6.log" 2>&1
