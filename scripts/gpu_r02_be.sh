#!/bin/bash
# L2 bulk prefetch of the next tile in k_dst4 / k_dst5 / k_tpass2 (default) vs none (CNPINT_L2PF=0): parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dst or timepass or c5 or c4 or pinv" > gpurun_out/pytest_pf.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_pf.log
rm -f gpurun_out/ab_pf.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n255_N1024 c4 c5_n511_N256; do
    for pf in 1 0; do
      echo "$wl pf=$pf $(CNPINT_L2PF=$pf timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_pf.txt
    done
  done
  for wl in c5_n511_N1024 c4; do
    for pf in 1 0; do
      echo "$wl pf=$pf gmres $(CNPINT_L2PF=$pf timeout 300 python scripts/gap_probe.py --workload $wl 2>&1 | tail -1)" >> gpurun_out/ab_pf.txt
    done
  done
done
echo done
