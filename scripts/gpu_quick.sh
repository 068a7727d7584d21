#!/bin/bash
# quick GPU check: selected parity tests + per-kernel timings
K=${1:-"pinv or stage or negative"}
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_quick.log
rm -f gpurun_out/times_quick.jsonl
for w in ${WL:-c1 c2 c3 c4}; do
  timeout 300 python scripts/prof_ops.py --workload $w --op pinv --reps 10 --time >> gpurun_out/times_quick.jsonl 2>> gpurun_out/times_quick.err
done
