#!/bin/bash
# K6 recurrence form (k_tscan) after the table-based closure: new tests, chunk-shape A/B, ncu --set full, whole GPU suite, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "timepass or negative_controls or dst_instantiations or pinv_full_c4 or pinv_small" > gpurun_out/pytest_tscan.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tscan.log
rm -f gpurun_out/ab_tscan2.txt
for wl in c5_n511_N1024 c4 c5_n511_N256; do
  for cfg in 16,8,2 8,16,2 16,8,3 8,8,4 4,16,2 16,16,1; do
    echo "$wl scan $cfg $(CNPINT_TSCAN_CFG=$cfg timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tscan2.txt
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tscan" -c 1 -o gpurun_out/prof_tscan -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_tscan.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_tscan.log
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
