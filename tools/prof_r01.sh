# ncu evidence for the round-1 kernels (text, small): per-config solve-kernel DRAM
# traffic + one detailed capture per top kernel of c1.  Outputs gpurun_out/n_*.
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread
for c in c1 c2 c3; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:lu_solve -c 2 --csv python tools/prof_op.py $c --apply prec --reps 1 > gpurun_out/n_solve_$c.csv 2>&1
done
SEC="--section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section ComputeWorkloadAnalysis --section LaunchStats"
timeout 600 ncu $SEC --clock-control none -k regex:"lu_solve_rag|zmul_shfl|fft_long2|reg_cols" --launch-skip 1 -c 6 --csv --page details python tools/prof_op.py c1 --apply both --reps 1 > gpurun_out/n_c1_details.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/n_c1_launches.csv 2>&1
ls -la gpurun_out/n_*
