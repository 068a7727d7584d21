#!/bin/bash
# lean 2D time pass (k_tpass2, debug 16384): parity + A/B + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass or negative" > gpurun_out/pytest_tp2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tp2.log
rm -f gpurun_out/ab_tp2.jsonl
for wl in c4 c5_n127_N256 c5_n127_N1024 c5_n255_N1024 c5_n511_N256 c5_n511_N1024; do
  for dbg in 0 16384; do
    echo "debug $dbg" >> gpurun_out/ab_tp2.jsonl
    timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg >> gpurun_out/ab_tp2.jsonl 2>> gpurun_out/ab_tp2.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tpass2" -c 1 -o gpurun_out/prof_tp2 -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 --debug 16384 > gpurun_out/ncu_tp2.log 2>&1
