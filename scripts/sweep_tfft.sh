#!/bin/bash
# time the time-FFT kernels for several cluster sizes C (CNPINT_TFFT_C override)
rm -f gpurun_out/sweep.jsonl
for w in c2 c4 c3 c1; do
for C in ${CS:-1 2 4 8}; do
  echo "{\"C\": $C, \"w\": \"$w\"}" >> gpurun_out/sweep.jsonl
  CNPINT_TFFT_C=$C timeout 120 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time >> gpurun_out/sweep.jsonl 2>>gpurun_out/sweep.err
done
done
