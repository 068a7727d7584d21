#!/bin/bash
# 2D time pass: the per-mode divide by a Newton-refined reciprocal (crecip_nr) instead of an IEEE division
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass or 2d or c4 or c5 or time_fft" > gpurun_out/pytest_div.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_div.log
rm -f gpurun_out/ab_div.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n255_N1024 c4 c5_n127_N256 c5_n511_N256; do
    echo "$wl new $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_div.txt
    echo "$wl old $(CNPINT_LIB=paper_2401_16113_b200/libcnpint_div0.so timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_div.txt
  done
done
echo done
