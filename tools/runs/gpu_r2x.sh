# round 2, call X: final R-MAT 27 numbers with the persisting window on the compact arrays: bench, launch list, ncu of both passes; R-MAT 24 bench
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2x
mkdir -p $OUT
KRE='regex:k1_|k_mark|k_cand|k_list|k_heavy|k_control|k_verify|k_census|k_class|k_check|k_graph'
( timeout 2400 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err; echo "rc=$?"
cut -c1-300 $OUT/bench_rmat27.json
GCOL_EAGER=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_rmat27.log 2>&1
for k in k1_heavy_wait k1_wait; do
  GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f \
    -o $OUT/$k python tools/one_run.py rmat27 > $OUT/ncu_$k.log 2>&1
  ( python tools/ncu_summary.py report $OUT/$k.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/$k.ncu-rep 20 ) > $OUT/${k}_rmat27_full.txt 2>&1
  rm -f $OUT/$k.ncu-rep
  head -8 $OUT/${k}_rmat27_full.txt
done
( timeout 1500 python bench.py --config rmat24 --steps 10 --warmup 3 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err; echo "rc=$?"
cut -c1-300 $OUT/bench_rmat24.json
