set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r27
mkdir -p $OUT
timeout 1200 python tools/compare_algorithms.py > $OUT/rsoc_vs_catalyurek.jsonl 2> $OUT/compare.err
timeout 2400 python bench.py --config rmat27 --steps 3 --warmup 3 --e2e-steps 3 --cpu-seconds 30 \
  > $OUT/bench_rmat27_full.json 2> $OUT/bench_rmat27_full.err
