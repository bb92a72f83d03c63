# round 2, call S: compact K1HW is bound by warp slots x latency (rows 17k, pieces 26k cycles): warps per SM, role split, piece batch
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2s
mkdir -p $OUT
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 3 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  echo "== $name"; tail -3 $OUT/probe_$name.log | cut -c1-420
}
probe w24_r16p8 rmat27
probe w24_r12p12 rmat27 GCOL_K1H_ROWW=12 GCOL_K1H_PIECEW=8
probe w32_r24p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_w32/libgcol_cuda.so
probe w32_r20p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_w32/libgcol_cuda.so GCOL_K1H_ROWW=20
probe pb16_r16p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_pb16/libgcol_cuda.so
probe w32pb16_r24p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_w32pb16/libgcol_cuda.so
