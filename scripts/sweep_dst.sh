#!/bin/bash
for w in c4 c5_n255_N1024; do
  for cfg in "" "CNPINT_LIB=paper_2401_16113_b200/libcnpint_d3.so"; do
    echo "$w $cfg $(env $cfg timeout 200 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time 2>&1 | tail -1)"
  done
done
