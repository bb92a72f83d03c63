# round 2, call N: K1HW with per-row claims and register-cached poll windows; 32-warp build; chain depth
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2n
mkdir -p $OUT
export GCOL_K1H_V=3 GCOL_K1_PROFILE=1 PROBE_VERIFY=0
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env "$@" timeout 600 python tools/class_probe.py $cfg 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-420
}
( timeout 600 python tools/hw_exact.py 16 20 ) > $OUT/exact.log 2>&1; tail -3 $OUT/exact.log | cut -c1-250
probe r24_default rmat24 PROBE_VERIFY=1
probe r24_rw8 rmat24 GCOL_K1H_ROWW=8
probe r24_rw20pw4 rmat24 GCOL_K1H_ROWW=20 GCOL_K1H_PIECEW=4
probe r24_w32 rmat24 GCOL_CUDA_LIB=$PWD/scratch_hw32/libgcol_cuda.so
probe r24_w32_pw4 rmat24 GCOL_CUDA_LIB=$PWD/scratch_hw32/libgcol_cuda.so GCOL_K1H_PIECEW=4 GCOL_K1H_ROWW=28
probe r27_default rmat27 GCOL_K1H_V=3
probe r27_w32 rmat27 GCOL_CUDA_LIB=$PWD/scratch_hw32/libgcol_cuda.so
( timeout 900 python tools/chain_depth.py rmat24 64 1024 ) > $OUT/chain_rmat24.log 2>&1; cat $OUT/chain_rmat24.log
