#!/bin/bash
# four-step FFT knobs at c2 / c3: lag, L2 discard, alternative builds (CNPINT_LIB)
for w in c2 c3; do
  for cfg in "" "CNPINT_FS_NODISCARD=1" "CNPINT_FS_LAG=24" "CNPINT_LIB=paper_2401_16113_b200/libcnpint_v4.so"; do
    echo "$w $cfg $(env $cfg timeout 120 python scripts/prof_ops.py --workload $w --op pinv --reps 10 --time 2>&1 | tail -1)"
  done
done
