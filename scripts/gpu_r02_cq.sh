#!/bin/bash
# residual launches (b - Mu with the norm) through the staged kernel (CNPINT_MVS_RES=1) vs the register kernel
mkdir -p gpurun_out
rm -f gpurun_out/ab_res.txt
for rep in 1 2; do
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  for r in 0 1; do
    echo "$wl res=$r $(CNPINT_MVS_RES=$r timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0 --reps 5 2>&1 | head -1)" >> gpurun_out/ab_res.txt
  done
done
done
for r in 0 1; do
  echo "c5_n511_N1024 res=$r $(CNPINT_MVS_RES=$r timeout 300 python scripts/prof_ops.py --workload c5_n511_N1024 --op gmres --reps 3 --time 2>&1 | tail -1)" >> gpurun_out/ab_res.txt
done
CNPINT_MVS_RES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "matvec2d_staged or gmres_small or gmres_restart or host_entry or gmres_c5_vs_oracle" > gpurun_out/pytest_res.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_res.log
