#!/bin/bash
# One gpurun call: GPU tests, per-kernel event timings per config, then ncu captures of the P^-1 kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for w in c2 c3 c4 c5_n511_N1024; do
  timeout 300 python scripts/prof_ops.py --workload $w --op all --reps 5 --time >> gpurun_out/times.jsonl 2>> gpurun_out/times.err
done
python scripts/prof_ops.py --workload c2 --op pinv --reps 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_tridiag|k_time_fft' -c 3 -o gpurun_out/prof_c2 -f \
    python scripts/prof_ops.py --workload c2 --op pinv --reps 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/prof_ops.py --workload c4 --op pinv --reps 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_dst|k_time_fft' -c 3 -o gpurun_out/prof_c4 -f \
    python scripts/prof_ops.py --workload c4 --op pinv --reps 1 > gpurun_out/ncu_c4.log 2>&1
echo done
