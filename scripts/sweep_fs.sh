#!/bin/bash
# K2 (four-step, c2) phase timing: CNPINT_FS_SKIP 1 = no input loads, 2 = no spectrum stores,
# 4 = no Y (L2) traffic; results wrong, timing only
for cfg in "" "CNPINT_FS_SKIP=1" "CNPINT_FS_SKIP=2" "CNPINT_FS_SKIP=4" "CNPINT_FS_SKIP=3" "CNPINT_FS_SKIP=7"; do
  echo "c2 $cfg $(env $cfg timeout 120 python scripts/prof_ops.py --workload c2 --op pinv --reps 10 --time 2>&1 | tail -1)"
done
