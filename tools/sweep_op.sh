#!/bin/bash
# parameter sweep of the FFT launch shapes (timing only)
for cfg in "4096 16 96 32" "8192 16 96 32" "4096 32 96 32" "4096 64 128 32" "4096 16 96 64" "4096 32 96 64" "16384 32 96 64" "2048 8 96 16"; do
  set -- $cfg
  VX_FFT_CONTIG_ELEMS=$1 VX_FFT_STRIDED_W=$2 VX_FFT_STRIDED_KB=$3 VX_ZMUL_W=$4 python tools/prof_op.py ${CONF:-c1} --reps 10 2>&1 | sed "s/^/[$cfg] /"
done
