# round 2, call V: ncu of the final R-MAT 27 kernels (compact light pass traffic; launch list of the bench command)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2v
mkdir -p $OUT
KRE='regex:k1_|k_mark|k_cand|k_list|k_heavy|k_control|k_verify|k_census|k_class|k_check|k_graph'
( timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ) > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
GCOL_EAGER=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_rmat27.log 2>&1
GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -f \
  -o $OUT/k1lc_rmat27 python tools/one_run.py rmat27 > $OUT/ncu_k1lc_rmat27.log 2>&1
( python tools/ncu_summary.py report $OUT/k1lc_rmat27.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/k1lc_rmat27.ncu-rep 20 ) > $OUT/k1l_compact_rmat27_full.txt 2>&1
rm -f $OUT/k1lc_rmat27.ncu-rep
head -12 $OUT/k1l_compact_rmat27_full.txt
