#!/bin/bash
for w in c5_n255_N1024 c5_n511_N1024; do
  for cfg in "" "CNPINT_FS_2D_MIN=1024" "CNPINT_FS_2D_MIN=1024 CNPINT_LIB=paper_2401_16113_b200/libcnpint_nc5_16.so" "CNPINT_FS_2D_MIN=1024 CNPINT_LIB=paper_2401_16113_b200/libcnpint_nc5_64.so"; do
    echo "$w $cfg $(env $cfg timeout 200 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time 2>&1 | tail -1)"
  done
done
