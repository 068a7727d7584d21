#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/gap.txt
for wl in c5_n511_N1024 c4 c2; do
  for pdl in 1 0; do
    CNPINT_PDL=$pdl timeout 300 python scripts/gap_probe.py --workload $wl >> gpurun_out/gap.txt 2>&1
  done
done
