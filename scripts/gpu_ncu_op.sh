#!/bin/bash
# usage: gpu_ncu_op.sh WORKLOAD KERNEL_REGEX TAG OP [LAUNCH_SKIP] -> ncu --set full of one launch of the kernel
W=$1; KRE=$2; TAG=$3; OP=$4; SKIP=${5:-0}
python scripts/prof_ops.py --workload $W --op $OP --reps 2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 -o gpurun_out/prof_$TAG -f \
    python scripts/prof_ops.py --workload $W --op $OP --reps 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
