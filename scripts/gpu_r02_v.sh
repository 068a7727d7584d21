#!/bin/bash
# k_tpass2 partner exchange by shuffles (N = 512, 1024) vs the previous build: parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass or c5 or 2d or c4 or dst" > gpurun_out/pytest_tp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tp.log
rm -f gpurun_out/ab_tp.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n127_N1024 c5_n255_N1024; do
    echo "$wl new $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
    echo "$wl old $(CNPINT_LIB=paper_2401_16113_b200/libcnpint_tp2old.so timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
  done
  echo "c4_512 new $(timeout 200 python scripts/prof_ops.py --workload c4 --op pinv --reps 5 --time --debug 16384 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
  echo "c4_512 old $(CNPINT_LIB=paper_2401_16113_b200/libcnpint_tp2old.so timeout 200 python scripts/prof_ops.py --workload c4 --op pinv --reps 5 --time --debug 16384 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
  echo "c4_def new $(timeout 200 python scripts/prof_ops.py --workload c4 --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
done
echo done
