# K1 timings on the resident BASELINE graphs, one process per environment
# setting (tooling; the graph exec is cached per handle), e.g.
#   ENVS="GCOL_K1W_SLEEP=0 GCOL_K1W_SLEEP=512" bash tools/k1w_sweep.sh
for env in ${ENVS:-NONE=1}; do
  env $env timeout 300 python tools/k1_ab.py ${CONFIGS:-tri er stencil} --variants 0 --runs 7 | sed "s/^{/{\"env\":\"$env\",/"
done
