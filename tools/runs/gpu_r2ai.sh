# round 2, call AI: the heavy-pass variants across R-MAT scales 16..23 (is the short poll budget a sane default below scale 24?)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ai
mkdir -p $OUT
( timeout 1200 python tools/scale_probe.py 16 18 20 22 23 ) > $OUT/scale_probe.log 2>&1; cat $OUT/scale_probe.log | cut -c1-200
