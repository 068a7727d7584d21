#!/bin/bash
# c3 four-step variants: FS_NC7 / FS_MINB7 builds via CNPINT_LIB
for cfg in "" "CNPINT_LIB=paper_2401_16113_b200/libcnpint_v8_4.so" "CNPINT_LIB=paper_2401_16113_b200/libcnpint_v8_3.so" "CNPINT_LIB=paper_2401_16113_b200/libcnpint_v16_3.so"; do
  echo "c3 $cfg $(env $cfg timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time 2>&1 | tail -1)"
done
