#!/bin/bash
# sine passes with the stage twiddles formed as powers in registers (libcnpint_twpow.so, -DDST_TWPOW) vs table reads
mkdir -p gpurun_out
rm -f gpurun_out/ab_twpow.txt
for rep in 1 2; do
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  echo "$wl base $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_twpow.txt
  echo "$wl twpow $(CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_twpow.so timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_twpow.txt
done
done
CNPINT_LIB=$PWD/paper_2401_16113_b200/libcnpint_twpow.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "dst or pinv_small or pinv_full_c4" > gpurun_out/pytest_twpow.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_twpow.log
