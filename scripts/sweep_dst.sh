#!/bin/bash
# K5: register DST (default routing) vs the shared-memory Stockham kernel everywhere (debug 32)
for w in c4 c5_n255_N1024; do
  for d in 0 32; do
    echo "$w $d $(timeout 200 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time --debug $d 2>&1 | tail -1)"
  done
done
