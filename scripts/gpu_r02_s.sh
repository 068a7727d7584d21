#!/bin/bash
# ncu --set full of the k_trivar solve launch at c3 (launch 0 of k_trivar is the per-handle table build)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_trivar" --launch-skip 1 -c 1 -o gpurun_out/prof_tv3s_c3 -f \
    python scripts/prof_ops.py --workload c3 --op pinv --reps 2 > gpurun_out/ncu_tv3s.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_tv3s.log
