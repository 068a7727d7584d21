#!/bin/bash
# K6 recurrence form (k_tscan): parity of the new tests, A/B against the transform kernels and across chunk shapes,
# then the whole GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "timepass or negative_controls or dst_instantiations or pinv_full_c4" > gpurun_out/pytest_tscan.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tscan.log
rm -f gpurun_out/ab_tscan.txt
for wl in c5_n511_N1024 c4 c5_n511_N256 c5_n127_N1024; do
  echo "$wl transform $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug 524288 2>&1 | tail -1)" >> gpurun_out/ab_tscan.txt
  echo "$wl scan default $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tscan.txt
  for cfg in 16,16 8,16 8,8 4,16; do
    echo "$wl scan $cfg $(CNPINT_TSCAN_CFG=$cfg timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tscan.txt
  done
done
for dbg in 524288 0; do
  timeout 300 python scripts/gap_probe.py --workload c5_n511_N1024 --debug $dbg 2>&1 | tail -1 | sed "s/^/debug $dbg /" >> gpurun_out/ab_tscan.txt
done
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
