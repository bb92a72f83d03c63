# round 2, call AH: R-MAT 24 end-to-end (streamed upload) against the heavy pass variant / poll budget
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ah
mkdir -p $OUT
run() { name=$1; shift
  ( env "$@" timeout 900 python bench.py --config rmat24 --steps 5 --warmup 3 --no-cpu-baseline ) > $OUT/bench_$name.json 2> $OUT/bench_$name.err
  python - <<PY
import json
d=json.loads(open("$OUT/bench_$name.json").read().strip().splitlines()[-1])
print("$name", "value", round(d["value"],1), "e2e", round(d["e2e"]["value"],2), round(d["e2e"]["ms_per_step"],1), "three-call", round(d["e2e"]["three_call_ms_per_step"],1), "rounds", d["colors"]["rounds"], d["colors"]["gpu_runs"])
PY
}
run default GCOL_X=0
run polls64 GCOL_K1H_POLLS=64
run exact GCOL_K1H_V=3
run spec GCOL_K1H_V=1
run default2 GCOL_X=0
