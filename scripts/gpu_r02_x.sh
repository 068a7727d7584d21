#!/bin/bash
# PDL: early trigger (default) vs trigger at exit (notrig build) vs off, on every BASELINE size class
mkdir -p gpurun_out
rm -f gpurun_out/gap2.txt
for wl in c5_n511_N1024 c5_n511_N256 c5_n255_N1024 c5_n127_N1024 c4 c3 c2; do
  CNPINT_PDL=1 timeout 300 python scripts/gap_probe.py --workload $wl >> gpurun_out/gap2.txt 2>&1
  CNPINT_PDL=0 timeout 300 python scripts/gap_probe.py --workload $wl >> gpurun_out/gap2.txt 2>&1
  CNPINT_LIB=paper_2401_16113_b200/libcnpint_notrig.so CNPINT_PDL=1 timeout 300 python scripts/gap_probe.py --workload $wl | sed 's/"pdl": "1"/"pdl": "notrig"/' >> gpurun_out/gap2.txt 2>&1
done
