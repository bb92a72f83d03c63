# round 2, call AB: where the R-MAT 27 end-to-end time goes (GCOL_TRACE phases of the one-call path, three calls)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ab
mkdir -p $OUT
( GCOL_TRACE=1 timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline ) > $OUT/bench_trace.json 2> $OUT/bench_trace.err; echo "rc=$?"
grep -E "gcol trace|color_rsoc_csr|^\[" $OUT/bench_trace.err | tail -40 | cut -c1-400
