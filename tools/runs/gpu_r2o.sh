# round 2, call O: K1HW integrated (k1_wide 6 / automatic above L2 size): new tests, full GPU suite, probes, R-MAT 27 bench
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2o
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "waiting or heavy_pass" ) > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
tail -5 $OUT/pytest_hw.log
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 600 python tools/class_probe.py $cfg 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-420
}
probe r24_wait rmat24 GCOL_K1H_V=3
probe r24_wait_rw8 rmat24 GCOL_K1H_V=3 GCOL_K1H_ROWW=8
probe r27_auto rmat27 PROBE_VERIFY=0
probe r27_w32 rmat27 GCOL_CUDA_LIB=$PWD/scratch_hw32/libgcol_cuda.so
( timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
( timeout 2400 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err; echo "rc=$?"
cut -c1-900 $OUT/bench_rmat27.json
