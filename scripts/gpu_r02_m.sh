#!/bin/bash
# K3 variable rows: coefficient-row prefetch A/B (c3) + tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "price or c3 or singular or tree" > gpurun_out/pytest_k3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k3.log
rm -f gpurun_out/ab_k3.jsonl
for i in 1 2; do
  timeout 300 python scripts/prof_ops.py --workload c3 --op pinv --reps 5 --time >> gpurun_out/ab_k3.jsonl 2>> gpurun_out/ab_k3.err
done
