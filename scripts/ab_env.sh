#!/bin/bash
# A/B of an environment knob on P^-1 kernel timings: AB_VAR=value pairs in $AB_SET (e.g. "CNPINT_TRI_F3=0 CNPINT_TRI_F3=1")
for rep in 1 2; do
  for kv in $AB_SET; do
    for w in ${AB_W:-c2}; do
      echo "$w $kv $(env $kv timeout 120 python scripts/prof_ops.py --workload $w --op ${AB_OP:-pinv} --reps 10 --time 2>&1 | tail -1)"
    done
  done
done
