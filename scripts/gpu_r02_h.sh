#!/bin/bash
# K5 / K6 compute-only timing (experiment build: CNPINT_DST_SKIP=1 no loads, 2 no stores, 3 neither)
mkdir -p gpurun_out
rm -f gpurun_out/dst_skip.jsonl
for wl in c4 c5_n511_N1024; do
  for sk in 0 1 2 3; do
    echo "skip $sk" >> gpurun_out/dst_skip.jsonl
    CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_ab.so CNPINT_DST_SKIP=$sk timeout 300 python scripts/prof_ops.py \
        --workload $wl --op pinv --reps 5 --time >> gpurun_out/dst_skip.jsonl 2>> gpurun_out/dst_skip.err
  done
done
