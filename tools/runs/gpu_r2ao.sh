# round 2, call AO: the three bounded-degree configs once more (no regression since round 1)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2ao
mkdir -p $OUT
for c in tri er stencil; do
  ( timeout 900 python bench.py --config $c ) > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "$c rc=$?"
  python - <<PY
import json
d=json.loads(open("$OUT/bench_$c.json").read().strip().splitlines()[-1])
print("$c", round(d["value"],1), "GE/s", round(d["ms_per_step"],4), "ms colours", d["colors"]["gpu"], "gate", d["colors"]["gate_1p05"], "rounds", d["colors"]["rounds"], "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"],2), "cpu", round(d["cpu_baseline"]["value"],2))
PY
done
