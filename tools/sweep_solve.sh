# A/B of the block-solve launch knobs (kprof per-kernel times)
for env in "" "VX_PIPE_BUDGET_KB=72" "VX_PIPE_BUDGET_KB=54" "VX_PIPE_BUDGET_KB=44" "VX_SECTORS=0" "VX_SECTORS=0 VX_PIPE_BUDGET_KB=150"; do
  echo "=== $env"; python tools/kprof.py ${CFG:-c1} --what prec --reps 5 --env $env X=1 2>&1 | grep -E "ms per step|lu_solve|sec_xform|fft_lines"
done
