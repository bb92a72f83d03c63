# round 2, call AK: role split of the waiting heavy pass at the short poll budget on R-MAT 24 (piece warps are 47 % busy)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ak
mkdir -p $OUT
for cfg in "16 8" "18 6" "20 4" "19 5"; do
  set -- $cfg
  ( GCOL_K1H_ROWW=$1 GCOL_K1H_PIECEW=$2 PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat24 5 0 ) > $OUT/probe_r$1p$2.log 2>&1
  echo "== row $1 piece $2"; tail -3 $OUT/probe_r$1p$2.log | cut -c1-200
done
