# round 2, call AE: waiting heavy pass with a small no-progress poll budget on R-MAT 24 (break the 4914-row chain by colouring past a stalled wait)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ae
mkdir -p $OUT
for p in 2 8 32 128 512; do
  ( GCOL_K1H_V=3 GCOL_K1H_POLLS=$p PROBE_VERIFY=0 timeout 600 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_polls$p.log 2>&1
  echo "== polls $p"; tail -3 $OUT/probe_polls$p.log | cut -c1-260
done
