#!/bin/bash
# k_tpass2 at N = 1024: 4 pairs per tile (two CTAs per SM) vs 8 (one CTA): parity with P = 4 + A/B
mkdir -p gpurun_out
CNPINT_TPASS2_P=4 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass or c5 or N1024" > gpurun_out/pytest_tp4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tp4.log
rm -f gpurun_out/ab_tp4.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n255_N1024 c5_n127_N1024; do
    for pp in 8 4; do
      echo "$wl P=$pp $(CNPINT_TPASS2_P=$pp timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tp4.txt
    done
  done
done
for pp in 8 4; do CNPINT_TPASS2_P=$pp timeout 300 python scripts/gap_probe.py --workload c5_n511_N1024 | sed "s/\"pdl\"/\"P\": $pp, \"pdl\"/" >> gpurun_out/ab_tp4.txt; done
echo done
