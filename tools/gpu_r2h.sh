# round 2, call H: benches after the class split + ncu evidence
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2h
mkdir -p $OUT
( timeout 900 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
( timeout 1200 python bench.py --steps 10 --warmup 3 ) > $OUT/bench_rmat27.json 2> $OUT/bench_rmat27.err
( timeout 900 python bench.py --config rmat24 --steps 10 --warmup 3 ) > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err
export GCOL_EAGER=1 PROBE_VERIFY=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_rmat24.csv python tools/class_probe.py rmat24 1 0 > $OUT/ncu_launches24.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_heavy -c 1 -o $OUT/k1h_rmat24 python tools/class_probe.py rmat24 1 0 > $OUT/ncu_k1h24.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_wait -c 1 -o $OUT/k1l_rmat24 python tools/class_probe.py rmat24 1 0 > $OUT/ncu_k1l24.log 2>&1
