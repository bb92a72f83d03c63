# round 2, call P: ncu evidence for the round-2 kernels.  Launch list of the default bench command
# (R-MAT 27, eager replay so the round kernels show), --set full captures of k1_heavy_wait and the
# light pass on R-MAT 27, of k1_heavy / k_list / k_heavy on R-MAT 24.  Each only after the plain run exited 0.
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2p
mkdir -p $OUT
KRE='regex:k1_|k_mark|k_cand|k_list|k_heavy|k_control|k_verify|k_census|k_class|k_check|k_graph'
( timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ) > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
GCOL_EAGER=1 timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_rmat27.log 2>&1
( timeout 600 python tools/one_run.py rmat27 ) > $OUT/one_rmat27.log 2>&1 && {
GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k1_heavy_wait -c 1 -f \
  -o $OUT/k1hw_rmat27 python tools/one_run.py rmat27 > $OUT/ncu_k1hw_rmat27.log 2>&1
GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -f \
  -o $OUT/k1l_rmat27 python tools/one_run.py rmat27 > $OUT/ncu_k1l_rmat27.log 2>&1
}
( timeout 600 python tools/one_run.py rmat24 ) > $OUT/one_rmat24.log 2>&1 && {
GCOL_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_heavy -c 1 -f \
  -o $OUT/k1h_rmat24 python tools/one_run.py rmat24 > $OUT/ncu_k1h_rmat24.log 2>&1
GCOL_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heavy -s 2 -c 1 -f \
  -o $OUT/kheavy_rmat24 python tools/one_run.py rmat24 > $OUT/ncu_kheavy_rmat24.log 2>&1
GCOL_EAGER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_list -c 1 -f \
  -o $OUT/klist_rmat24 python tools/one_run.py rmat24 > $OUT/ncu_klist_rmat24.log 2>&1
GCOL_EAGER=1 GCOL_K1H_V=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_heavy_wait -c 1 -f \
  -o $OUT/k1hw_rmat24 python tools/one_run.py rmat24 > $OUT/ncu_k1hw_rmat24.log 2>&1
GCOL_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 400 --csv \
  --log-file $OUT/launches_rmat24.csv python tools/one_run.py rmat24 > $OUT/launches_rmat24.log 2>&1
}
# summaries here (the reports together exceed what gpurun brings back); one report kept
for r in k1hw_rmat27 k1l_rmat27 k1h_rmat24 kheavy_rmat24 klist_rmat24 k1hw_rmat24; do
  if [ -f $OUT/$r.ncu-rep ]; then
    ( python tools/ncu_summary.py report $OUT/$r.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/$r.ncu-rep 20 ) > $OUT/${r}_full.txt 2>&1
    [ $r = k1hw_rmat27 ] || rm -f $OUT/$r.ncu-rep
  fi
done
ls -la $OUT
