#!/bin/bash
# k_tpass2 GEN 2 (cp.async prefetch + table divide) vs GEN 1 (debug 262144): parity + per-launch A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass or c5 or mesh or c4" > gpurun_out/pytest_tp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tp.log
rm -f gpurun_out/ab_tp.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n255_N1024 c5_n127_N256 c5_n511_N256; do
    for dbg in 0 262144; do
      echo "$wl dbg=$dbg $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg 2>&1 | tail -1)" >> gpurun_out/ab_tp.txt
    done
  done
done
echo done
