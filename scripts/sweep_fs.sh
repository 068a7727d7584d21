#!/bin/bash
for w in c2 c3; do
    echo "$w $(timeout 120 python scripts/prof_ops.py --workload $w --op pinv --reps 10 --time 2>&1 | tail -1)"
done
