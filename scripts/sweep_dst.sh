#!/bin/bash
for w in c4; do
  for d in 0 128; do
    echo "$w $d $(timeout 200 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time --debug $d 2>&1 | tail -1)"
  done
done
