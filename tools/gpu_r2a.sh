# round 2, call A: gpu tests + default bench (rmat27) + reference arm timing
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2a
mkdir -p $OUT
nproc > $OUT/host.txt; free -g >> $OUT/host.txt; lscpu | head -20 >> $OUT/host.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > $OUT/bench_default.json 2> $OUT/bench_default.err
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/bench_ref.json 2> $OUT/bench_ref.err
