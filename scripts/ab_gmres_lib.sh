#!/bin/bash
# GMRES time-to-tolerance, default library vs $AB_LIB, alternating twice (scripts/gmres_ab.py, debug 0)
for rep in 1 2; do
  for lib in "" "$AB_LIB"; do
    if [ -n "$lib" ]; then export CNPINT_LIB=$lib; else unset CNPINT_LIB; fi
    python scripts/gmres_ab.py --workloads ${AB_W:-c2,c3,c4} --debugs 0 | grep '"ms"' | sed "s|^|${lib:-default} |"
  done
done
