# A/B of the block-solve launch knobs (kprof per-kernel times)
for env in ${ENVS:-"" "VX_PIPE_BUDGET_KB=60" "VX_PIPE_BUDGET_KB=66" "VX_PIPE_BUDGET_KB=80" "VX_PIPE_BUDGET_KB=90"}; do
  echo "=== $env"; python tools/kprof.py ${CFG:-c1} --what prec --reps 5 --env $env X=1 2>&1 | grep -E "ms per step|lu_solve"
done
