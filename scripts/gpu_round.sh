#!/bin/bash
# One gpurun call: all GPU tests, the bench + its launch list, then ncu --set full of the hot kernels.
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
bash scripts/gpu_bench.sh
rm -f gpurun_out/times.jsonl
for w in c1 c2 c3 c4 c5_n511_N1024; do
  timeout 300 python scripts/prof_ops.py --workload $w --op all --reps 5 --time >> gpurun_out/times.jsonl 2>> gpurun_out/times.err
done
bash scripts/gpu_ncu_env.sh c2 "k_fstep" full_c2_k2 X=1
bash scripts/gpu_ncu_env.sh c2 "k_tridiag" full_c2_k3 X=1
bash scripts/gpu_ncu_env.sh c4 "k_dst" full_c4_k5 X=1
bash scripts/gpu_ncu_env.sh c4 "k_tpass" full_c4_k6 X=1
bash scripts/gpu_ncu_env.sh c3 "k_tridiag" full_c3_k3 X=1
bash scripts/gpu_ncu_op.sh c2 "k_update" full_c2_k7 gmres 3
bash scripts/gpu_ncu_env.sh c3 "k_fstep" full_c3_k2 X=1
bash scripts/gpu_ncu_op.sh c2 "k_matvec1d" full_c2_k1 A 0
bash scripts/gpu_ncu_op.sh c2 "k_matvec1d" full_c2_k1g gmres 1
bash scripts/gpu_ncu_env.sh c4 "k_dst_r" full_c4_k5y X=1
echo done
