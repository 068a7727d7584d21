#!/bin/bash
# K2/K4 at c3 (k_fstep<.,7,7>): default (2 CTAs/SM, 128 registers, spills) vs 1 CTA/SM (no spills) vs 8-pair blocks
mkdir -p gpurun_out
rm -f gpurun_out/fs7.jsonl
for lib in default fsminb1 fsnc8; do
  L=""; [ "$lib" != default ] && L=$PWD/paper_2401_16113_b200/libcnpint_$lib.so
  for wl in c3; do
    echo "lib $lib" >> gpurun_out/fs7.jsonl
    CNPINT_LIB=$L timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time >> gpurun_out/fs7.jsonl 2>> gpurun_out/fs7.err
    CNPINT_LIB=$L timeout 300 python scripts/prof_ops.py --workload $wl --op gmres --reps 3 --time >> gpurun_out/fs7.jsonl 2>> gpurun_out/fs7.err
  done
done
