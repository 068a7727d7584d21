#!/bin/bash
# source-level stall profile of the headline's sine passes
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dst4|k_dst5" -c 2 -o gpurun_out/prof_c5h -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_c5h.log 2>&1
echo "ncu c5h exit $?" >> gpurun_out/ncu_c5h.log
