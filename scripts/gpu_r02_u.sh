#!/bin/bash
# k_trivar with the create-time constants loaded before griddepcontrol.wait: parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_variable or price or c3 or singular or P1 or stage or tv" > gpurun_out/pytest_tv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tv.log
rm -f gpurun_out/ab_tv.txt
for rep in 1 2; do
  echo "pre-pdl $(timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
  echo "gmres $(timeout 120 python scripts/prof_ops.py --workload c3 --op gmres --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
done
echo done
