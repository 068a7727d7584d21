#!/bin/bash
# cache-policy experiment: evict-first (.cs) loads/stores vs default policy (CNPINT_LIB builds)
for lib in "" "paper_2401_16113_b200/libcnpint_l2L.so" "paper_2401_16113_b200/libcnpint_l2S.so" "paper_2401_16113_b200/libcnpint_l2LS.so"; do
  for w in c2 c4; do
    if [ -n "$lib" ]; then export CNPINT_LIB=$lib; else unset CNPINT_LIB; fi
    echo "$w ${lib:-default} $(python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-streams 1 2>/dev/null | tail -1)"
  done
done
