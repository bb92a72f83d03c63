set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r27
mkdir -p $OUT
free -g > $OUT/free.txt; nproc >> $OUT/free.txt
GCOL_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_tri_eager.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > $OUT/launches_tri.log 2>&1
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> $OUT/mem.txt; sleep 2; done ) &
MP=$!
timeout 1500 python bench.py --config rmat27 --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline \
  > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err
kill $MP
