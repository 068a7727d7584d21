#!/bin/bash
# GMRES time-to-tolerance with an environment knob toggled (AB_SET pairs), alternating twice
for rep in 1 2; do
  for kv in $AB_SET; do
    env $kv python scripts/gmres_ab.py --workloads ${AB_W:-c2,c3,c4} --debugs 0 | grep '"ms"' | sed "s|^|$kv |"
  done
done
