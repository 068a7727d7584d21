#!/bin/bash
# k_dst5 (y sine pass): 4 column pairs per tile with four CTAs per SM (libcnpint_d5p4.so), L2 prefetch of the next tile (CNPINT_D5_PF=1)
mkdir -p gpurun_out
rm -f gpurun_out/ab_d5.txt
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  echo "$wl base $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_d5.txt
  echo "$wl pf $(CNPINT_D5_PF=1 timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_d5.txt
  echo "$wl p4 $(CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_d5p4.so timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_d5.txt
  echo "$wl p4pf $(CNPINT_D5_PF=1 CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_d5p4.so timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_d5.txt
done
CNPINT_D5_PF=1 CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_d5p4.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "dst or pinv_small or pinv_full_c4" > gpurun_out/pytest_d5.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_d5.log
