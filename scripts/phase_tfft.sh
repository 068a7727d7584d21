#!/bin/bash
rm -f gpurun_out/phase.jsonl
for C in 2 4 8; do
for sk in 0 1 2 3; do
  echo "{\"skip\": $sk, \"C\": $C}" >> gpurun_out/phase.jsonl
  CNPINT_TFFT_C=$C CNPINT_TFFT_SKIP=$sk timeout 120 python scripts/prof_ops.py --workload c2 --op pinv --reps 5 --time >> gpurun_out/phase.jsonl 2>>gpurun_out/phase.err
done
done
