#!/bin/bash
# fused x+y sine pass (k_dstxy): parity + A/B (debug 0 fused vs 32768 five passes) + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dst or negative or timepass or c4 or c5" > gpurun_out/pytest_xy.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_xy.log
rm -f gpurun_out/ab_xy.jsonl
for wl in c4 c5_n127_N1024 c5_n255_N1024 c5_n511_N1024; do
  for dbg in 0 32768; do
    echo "debug $dbg" >> gpurun_out/ab_xy.jsonl
    timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg >> gpurun_out/ab_xy.jsonl 2>> gpurun_out/ab_xy.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dstxy" -c 2 -o gpurun_out/prof_xy -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_xy.log 2>&1
