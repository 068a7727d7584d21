#!/bin/bash
# register 2D matvec with fused dots: time rows per block (CNPINT_MV2_TCHUNK applies to every 2D matvec launch)
mkdir -p gpurun_out
rm -f gpurun_out/ab_mv2tc.txt
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  for tc in 16 32 64; do
    echo "$wl tchunk=$tc gmres $(CNPINT_MV2_TCHUNK=$tc timeout 300 python scripts/prof_ops.py --workload $wl --op gmres --reps 3 --time 2>&1 | tail -1)" >> gpurun_out/ab_mv2tc.txt
    echo "$wl tchunk=$tc $(CNPINT_MV2_TCHUNK=$tc timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0 --reps 5 2>&1 | head -1)" >> gpurun_out/ab_mv2tc.txt
  done
done
