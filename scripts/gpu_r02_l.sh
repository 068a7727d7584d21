#!/bin/bash
# SASS-level ncu captures of the 1D P^-1 kernels (c2, c3) and the N = 512 time pass (c4)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fstep|k_tridiag" -c 3 -o gpurun_out/prof_c2_1d -f \
    python scripts/prof_ops.py --workload c2 --op pinv --reps 1 > gpurun_out/ncu_c2_1d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fstep|k_tridiag" -c 3 -o gpurun_out/prof_c3_1d -f \
    python scripts/prof_ops.py --workload c3 --op pinv --reps 1 > gpurun_out/ncu_c3_1d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tpass" -c 1 -o gpurun_out/prof_c4_tp -f \
    python scripts/prof_ops.py --workload c4 --op pinv --reps 1 > gpurun_out/ncu_c4_tp.log 2>&1
