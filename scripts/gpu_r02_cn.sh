#!/bin/bash
# k_tscan: cluster scheduling policy (CNPINT_TSCAN_POL 1 = spread, 2 = load balancing) and the number of co-resident clusters
mkdir -p gpurun_out
rm -f gpurun_out/ab_tspol.txt
CNPINT_TSCAN_INFO=1 timeout 200 python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 2>&1 | grep tscan | head -2 >> gpurun_out/ab_tspol.txt
for wl in c5_n511_N1024 c4; do
  for pol in 0 1 2; do
    echo "$wl pol=$pol $(CNPINT_TSCAN_POL=$pol timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tspol.txt
  done
done
