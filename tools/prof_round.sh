# ncu captures for the op / prec kernels of one workload (usage: CFG=c1 bash tools/prof_round.sh)
set -x
CFG=${CFG:-c1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-fft_lines|zmul|reg_cols|lu_solve_pipe}" -c ${NCAP:-8} -o gpurun_out/p_${CFG}_full python tools/prof_op.py $CFG --apply ${APPLY:-both} --reps 1 > gpurun_out/p_${CFG}_ncu.log 2>&1
ls -la gpurun_out
