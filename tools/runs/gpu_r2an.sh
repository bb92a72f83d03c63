# round 2, call AN: ncu --set full of the default R-MAT 24 heavy pass (waiting, poll budget 6, 18 + 6 warps) and its light pass
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2an
mkdir -p $OUT
( timeout 600 python tools/one_run.py rmat24 ) > $OUT/one_rmat24.log 2>&1 && \
for k in k1_heavy_wait k1_wait; do
  GCOL_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f \
    -o $OUT/$k python tools/one_run.py rmat24 > $OUT/ncu_$k.log 2>&1
  ( python tools/ncu_summary.py report $OUT/$k.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/$k.ncu-rep 20 ) > $OUT/${k}_rmat24_full.txt 2>&1
  rm -f $OUT/$k.ncu-rep
  head -8 $OUT/${k}_rmat24_full.txt
done
