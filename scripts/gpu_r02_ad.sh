#!/bin/bash
# Gram update fused with the next x sine pass (k_upd_dst4): parity + A/B (debug 131072 = separate kernels) + ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fused_with_x or gmres or c4 or c5 or 2d" > gpurun_out/pytest_ud.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ud.log
rm -f gpurun_out/ab_ud.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n511_N256 c5_n255_N1024 c4 c5_n127_N1024; do
    for dbg in 0 131072; do
      timeout 300 python scripts/gap_probe.py --workload $wl --debug $dbg >> gpurun_out/ab_ud.txt 2>&1
    done
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_upd_dst4" -c 2 -o gpurun_out/prof_ud -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op gmres --reps 1 > gpurun_out/ncu_ud.log 2>&1
echo done
