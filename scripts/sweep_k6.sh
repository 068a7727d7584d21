#!/bin/bash
# K6 2D time pass: default routing (register kernel at N = 256/512) vs cluster kernel (debug 64)
for w in c4 c5_n255_N1024 c5_n511_N1024; do
  for d in 0 64; do
    echo "$w $d $(timeout 200 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time --debug $d 2>&1 | tail -1)"
  done
done
