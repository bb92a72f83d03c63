# Bench lines for the four single-GPU configs into gpurun_out/benches (tooling)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/benches
for c in ${CONFIGS:-tri er stencil rmat24}; do
  timeout 600 python bench.py --config $c > gpurun_out/benches/bench_$c.json 2> gpurun_out/benches/bench_$c.err
done
