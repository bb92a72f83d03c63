# round 2, call AF: poll budget of the waiting heavy pass, finer on R-MAT 24, and on R-MAT 27
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2af
mkdir -p $OUT
nvidia-smi --query-gpu=name,uuid,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
for p in 4 6 8 12 16 24; do
  ( GCOL_K1H_V=3 GCOL_K1H_POLLS=$p PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat24 5 0 ) > $OUT/probe24_polls$p.log 2>&1
  echo "== rmat24 polls $p"; tail -5 $OUT/probe24_polls$p.log | cut -c1-200
done
for p in 8 32 128; do
  ( GCOL_K1H_POLLS=$p PROBE_VERIFY=0 timeout 900 python tools/class_probe.py rmat27 3 0 ) > $OUT/probe27_polls$p.log 2>&1
  echo "== rmat27 polls $p"; tail -3 $OUT/probe27_polls$p.log | cut -c1-200
done
