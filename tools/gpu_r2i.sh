# round 2, call I (re-entry): confirm HEAD on a fresh box: tests, smoke, headline benches, reference arm
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2i
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
( timeout 1200 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
( timeout 1500 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err
( timeout 900 python bench.py --config rmat24 --steps 10 --warmup 3 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err
( timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 ) > $OUT/bench_reference_rmat27.json 2> $OUT/bench_reference_rmat27.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log | tail -2; cat $OUT/bench_*.json
