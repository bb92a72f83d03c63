# round 2, call U: light pass reading heavy colours through the compact array: tests, A/B on R-MAT 27, full suite, bench
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2u
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "waiting or heavy_pass or class_split" ) > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
tail -5 $OUT/pytest_hw.log
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 3 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  echo "== $name"; tail -3 $OUT/probe_$name.log | cut -c1-330
}
probe r27_lcompact rmat27 PROBE_VERIFY=1
probe r27_hcompact_only rmat27 GCOL_K1L_COMPACT=0
( timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
( timeout 2400 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err; echo "rc=$?"
cut -c1-400 $OUT/bench_rmat27.json
