# round 2, call AJ: where the R-MAT 24 heavy pass spends its time at poll budgets 2 / 6 / exact (GCOL_K1_PROFILE)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2aj
mkdir -p $OUT
for p in 2 6 4194304; do
  ( GCOL_K1_PROFILE=1 GCOL_K1H_POLLS=$p PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat24 3 0 ) > $OUT/probe_polls$p.log 2>&1
  echo "== polls $p"; tail -2 $OUT/probe_polls$p.log | cut -c1-420
done
