# round 2, call J: k1_heavy2 (decoupled K1H) -- correctness subset, then A/B and knob sweep on R-MAT 24
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2j
mkdir -p $OUT
( timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "class or heavy or rmat or split or stream" ) > $OUT/pytest_subset.log 2>&1; echo "rc=$?" >> $OUT/pytest_subset.log
tail -3 $OUT/pytest_subset.log
export GCOL_K1_PROFILE=1
probe() { # name, env...
  name=$1; shift
  ( env "$@" timeout 300 python tools/class_probe.py rmat24 4 0 ) > $OUT/probe_$name.log 2>&1; echo "rc=$?" >> $OUT/probe_$name.log
  tail -4 $OUT/probe_$name.log | cut -c1-400
}
probe v2_default GCOL_K1H_V=2
probe v1 GCOL_K1H_V=1 PROBE_VERIFY=0
probe v2_cw2 GCOL_K1H_CW=2 PROBE_VERIFY=0
probe v2_cw8 GCOL_K1H_CW=8 GCOL_K1H_PIECEW=6 PROBE_VERIFY=0
probe v2_cw1 GCOL_K1H_CW=1 PROBE_VERIFY=0
probe v2_polls4 GCOL_K1H_POLLS=4 PROBE_VERIFY=0
probe v2_polls32 GCOL_K1H_POLLS=32 PROBE_VERIFY=0
probe v2_ring16 GCOL_K1H_RING=16 PROBE_VERIFY=0
probe v2_ring32 GCOL_K1H_RING=32 PROBE_VERIFY=0
probe v2_pw4 GCOL_K1H_PIECEW=4 PROBE_VERIFY=0
probe v2_bps2 GCOL_K1H_BPS=2 PROBE_VERIFY=0
