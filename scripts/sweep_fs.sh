#!/bin/bash
for w in c2; do
  for cfg in "" "CNPINT_FS_SKIP=7"; do
    echo "$w $cfg $(env $cfg timeout 120 python scripts/prof_ops.py --workload $w --op pinv --reps 10 --time 2>&1 | tail -1)"
  done
done
