# round 2, call R: compact heavy colours inside K1HW (rank table + colours by rank): tests, then A/B on R-MAT 27 and 24
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2r
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "waiting or heavy_pass or class_split" ) > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
tail -5 $OUT/pytest_hw.log
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-420
}
probe r27_compact rmat27 PROBE_VERIFY=1
probe r27_plain rmat27 GCOL_K1HW_COMPACT=0
probe r24_compact rmat24 GCOL_L2_COLOURS_MB=0
probe r24_plain rmat24 GCOL_K1H_V=3
