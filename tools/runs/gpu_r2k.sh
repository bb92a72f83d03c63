# round 2, call K: bisect the R-MAT 24 K1H regression (4.6 -> 5.9 ms) over three older builds; v1 default restored
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2k
mkdir -p $OUT
export GCOL_K1_PROFILE=1 PROBE_VERIFY=0
for c in d83440b 686dd9b d30269f head; do
  lib=scratch_bisect/$c/libgcol_cuda.so; [ $c = head ] && lib=paper_1505_04086_b200/libgcol_cuda.so
  ( GCOL_CUDA_LIB=$PWD/$lib timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_$c.log 2>&1; echo "rc=$?" >> $OUT/probe_$c.log
  tail -3 $OUT/probe_$c.log | cut -c1-300
done
( GCOL_K1_PROFILE= timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_head_noprof.log 2>&1
tail -3 $OUT/probe_head_noprof.log | cut -c1-300
( GCOL_CUDA_LIB=$PWD/scratch_bisect/d83440b/libgcol_cuda.so GCOL_K1_PROFILE= timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_d83440b_noprof.log 2>&1
tail -3 $OUT/probe_d83440b_noprof.log | cut -c1-300
