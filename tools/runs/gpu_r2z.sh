# round 2, call Z: full validation of the final tree on a fresh box: GPU suite, smoke, default bench, reference arm
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2z
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
( timeout 1800 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log; cat $OUT/smoke.log
( timeout 2400 python bench.py ) > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "rc=$?"
cut -c1-260 $OUT/bench_default.json
( timeout 1800 python bench.py --impl reference ) > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "rc=$?"
cut -c1-400 $OUT/bench_reference.json
( timeout 120 python bench.py --gpus 2 --steps 2 --warmup 1 ) > $OUT/bench_gpus2.log 2>&1; echo "gpus2 rc=$?"; tail -2 $OUT/bench_gpus2.log | cut -c1-200
