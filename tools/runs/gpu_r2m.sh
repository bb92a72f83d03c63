# round 2, call M: K1HW (waiting heavy pass, GCOL_K1H_V=3): exactness on small R-MATs, then R-MAT 24 probes and knobs, R-MAT 27
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2m
mkdir -p $OUT
export GCOL_K1H_V=3
( timeout 600 python tools/hw_exact.py 14 16 18 20 ) > $OUT/exact.log 2>&1; echo "rc=$?" >> $OUT/exact.log
tail -14 $OUT/exact.log | cut -c1-300
export GCOL_K1_PROFILE=1
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env "$@" timeout 600 python tools/class_probe.py $cfg 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-420
}
probe r24_default rmat24 GCOL_K1H_V=3
probe r24_rw8 rmat24 GCOL_K1H_ROWW=8 PROBE_VERIFY=0
probe r24_rw20pw4 rmat24 GCOL_K1H_ROWW=20 GCOL_K1H_PIECEW=4 PROBE_VERIFY=0
probe r24_rw12 rmat24 GCOL_K1H_ROWW=12 PROBE_VERIFY=0
probe r27_default rmat27 PROBE_VERIFY=0
