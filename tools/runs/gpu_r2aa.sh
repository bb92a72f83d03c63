# round 2, call AA: GPU suite + R-MAT probes after removing k1_heavy2
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2aa
mkdir -p $OUT
( timeout 1800 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
( PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat24 3 0 ) > $OUT/probe_rmat24.log 2>&1; tail -1 $OUT/probe_rmat24.log | cut -c1-200
( PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat27 3 0 ) > $OUT/probe_rmat27.log 2>&1; tail -1 $OUT/probe_rmat27.log | cut -c1-200
