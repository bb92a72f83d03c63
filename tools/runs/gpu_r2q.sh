# round 2, call Q: K1HW hop latency (poll window fixed while the position moves inside it; slot bitmap read before the wait): A/B against the previous build
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2q
mkdir -p $OUT
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 600 python tools/class_probe.py $cfg 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-420
}
( GCOL_K1H_V=3 timeout 600 python tools/hw_exact.py 16 20 ) > $OUT/exact.log 2>&1; tail -2 $OUT/exact.log | cut -c1-250
probe r24_before rmat24 GCOL_K1H_V=3 GCOL_CUDA_LIB=$PWD/scratch_hwopt/libgcol_cuda_before.so
probe r24_after rmat24 GCOL_K1H_V=3
probe r24_after_rw8 rmat24 GCOL_K1H_V=3 GCOL_K1H_ROWW=8
probe r27_before rmat27 GCOL_CUDA_LIB=$PWD/scratch_hwopt/libgcol_cuda_before.so
probe r27_after rmat27 PROBE_VERIFY=0
