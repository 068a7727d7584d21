#!/bin/bash
# register 2D matvec: batches of 2 time rows also with 4-5 dot vectors (libcnpint_tbx.so, -DMV2D_TBX) vs 1
mkdir -p gpurun_out
rm -f gpurun_out/ab_tbx.txt
for rep in 1 2; do
for wl in c5_n511_N1024 c4; do
  echo "$wl base $(timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0 --reps 5 2>&1 | head -1)" >> gpurun_out/ab_tbx.txt
  echo "$wl tbx $(CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_tbx.so timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0 --reps 5 2>&1 | head -1)" >> gpurun_out/ab_tbx.txt
done
done
echo "base $(timeout 300 python scripts/prof_ops.py --workload c5_n511_N1024 --op gmres --reps 3 --time 2>&1 | tail -1)" >> gpurun_out/ab_tbx.txt
echo "tbx $(CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_tbx.so timeout 300 python scripts/prof_ops.py --workload c5_n511_N1024 --op gmres --reps 3 --time 2>&1 | tail -1)" >> gpurun_out/ab_tbx.txt
