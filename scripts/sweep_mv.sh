#!/bin/bash
for w in c2 c3 c4; do
  echo "$w $(timeout 200 python scripts/prof_ops.py --workload $w --op all --reps 5 --time 2>&1 | tail -1)"
done
