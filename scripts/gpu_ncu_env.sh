#!/bin/bash
# usage: gpu_ncu_env.sh WORKLOAD KERNEL_REGEX TAG [ENV...] -> ncu capture with environment overrides
W=$1; KRE=$2; TAG=$3; shift 3
env "$@" python scripts/prof_ops.py --workload $W --op pinv --reps 2 > gpurun_out/plain_$TAG.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 -o gpurun_out/prof_$TAG -f \
    python scripts/prof_ops.py --workload $W --op pinv --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
