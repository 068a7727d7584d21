#!/bin/bash
# lean x pass (k_dst4, debug 4096): parity + A/B timing + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dst_paths or dst_instantiations or negative" > gpurun_out/pytest_dst45.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dst45.log
rm -f gpurun_out/ab_dst45.jsonl
for wl in c4 c5_n127_N1024 c5_n255_N1024 c5_n511_N1024; do
  for dbg in 0 12288; do
    echo "debug $dbg" >> gpurun_out/ab_dst45.jsonl
    timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg >> gpurun_out/ab_dst45.jsonl 2>> gpurun_out/ab_dst45.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dst4" -c 1 -o gpurun_out/prof_dst4 -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_dst4.log 2>&1
