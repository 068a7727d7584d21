#!/bin/bash
# ncu --set full (source) of the headline's sine passes and time pass after GEN 2, plus c2's four-step K2/K4
mkdir -p gpurun_out
python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dst4|k_dst5|k_tpass2" -c 3 -o gpurun_out/prof_c5h -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_c5h.log 2>&1
echo "ncu c5h exit $?" >> gpurun_out/ncu_c5h.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fstep" -c 2 -o gpurun_out/prof_c2fs -f \
    python scripts/prof_ops.py --workload c2 --op pinv --reps 1 > gpurun_out/ncu_c2fs.log 2>&1
echo "ncu c2 exit $?" >> gpurun_out/ncu_c2fs.log
