#!/bin/bash
# k_matvec2d: 3 blocks per SM (MV2D_MINB=3 build, spills) vs 2 (default): per-class times in a GMRES solve
mkdir -p gpurun_out
rm -f gpurun_out/ab_mv.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c4 c5_n255_N1024; do
    echo "$wl mv2 $(timeout 300 python scripts/gap_probe.py --workload $wl 2>&1 | tail -1)" >> gpurun_out/ab_mv.txt
    echo "$wl mv3 $(CNPINT_LIB=paper_2401_16113_b200/libcnpint_mv3.so timeout 300 python scripts/gap_probe.py --workload $wl 2>&1 | tail -1)" >> gpurun_out/ab_mv.txt
  done
done
echo done
