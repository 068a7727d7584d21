#!/bin/bash
# A/B: default library vs $AB_LIB (same box), alternating, workloads in $AB_W (default c2 c4)
for rep in 1 2; do
for lib in "" "$AB_LIB"; do
  for w in ${AB_W:-c2 c4}; do
    if [ -n "$lib" ]; then export CNPINT_LIB=$lib; else unset CNPINT_LIB; fi
    echo "$w ${lib:-default} $(python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-streams 1 2>/dev/null | tail -1)"
  done
done
done
