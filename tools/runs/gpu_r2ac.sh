# round 2, call AC: K1HW micro-optimisations (batch records staged by the claimer, release reduction at the end of a piece): A/B + tests
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ac
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "waiting or heavy_pass or class_split" ) > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
tail -3 $OUT/pytest_hw.log
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 3 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  echo "== $name"; tail -3 $OUT/probe_$name.log | cut -c1-330
}
probe r27_before rmat27 GCOL_CUDA_LIB=$PWD/scratch_before/libgcol_cuda.so
probe r27_after rmat27 PROBE_VERIFY=1
probe r24w_before rmat24 GCOL_K1H_V=3 GCOL_CUDA_LIB=$PWD/scratch_before/libgcol_cuda.so
probe r24w_after rmat24 GCOL_K1H_V=3
