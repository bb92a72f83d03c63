# round 2, call W: L2 persisting window over rank table + heavy colours (one allocation) in the compact path
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2w
mkdir -p $OUT
python - <<'PY' > $OUT/l2_attrs.txt 2>&1
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size)
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if False else None
PY
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "compact or waiting" ) > $OUT/pytest_hw.log 2>&1; echo "rc=$?" >> $OUT/pytest_hw.log
tail -3 $OUT/pytest_hw.log
probe() { # name cfg env...
  name=$1; cfg=$2; shift; shift
  ( env GCOL_K1_PROFILE=1 PROBE_VERIFY=0 "$@" timeout 900 python tools/class_probe.py $cfg 3 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  echo "== $name"; tail -3 $OUT/probe_$name.log | cut -c1-330
}
probe r27_window rmat27
probe r27_nowindow rmat27 GCOL_L2_PERSIST=0
