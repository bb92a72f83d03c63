# round 2, call Y: role split / warps per SM again, now that the compact arrays own the L2
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2y
mkdir -p $OUT
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 3 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  echo "== $name"; tail -3 $OUT/probe_$name.log | cut -c1-330
}
probe w24_r16p8 rmat27
probe w24_r14p10 rmat27 GCOL_K1H_ROWW=14 GCOL_K1H_PIECEW=8
probe w32_r24p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_w32/libgcol_cuda.so
probe w32_r20p8 rmat27 GCOL_CUDA_LIB=$PWD/scratch_w32/libgcol_cuda.so GCOL_K1H_ROWW=20
for k in k1_heavy_wait k1_wait; do
  GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f \
    -o $OUT/$k python tools/one_run.py rmat27 > $OUT/ncu_$k.log 2>&1
  ( python tools/ncu_summary.py report $OUT/$k.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/$k.ncu-rep 20 ) > $OUT/${k}_rmat27_full.txt 2>&1
  rm -f $OUT/$k.ncu-rep
  head -8 $OUT/${k}_rmat27_full.txt
done
GCOL_EAGER=1 GCOL_K1_PROFILE=1 timeout 600 python tools/one_run.py rmat27 > $OUT/eager_rmat27.log 2>&1; tail -2 $OUT/eager_rmat27.log | cut -c1-300
