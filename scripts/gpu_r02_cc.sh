#!/bin/bash
# K6 recurrence form (k_tscan) in rho-minus-one form, relaxed cluster arrives: whole GPU suite, smoke, timings, ncu, bench.
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
rm -f gpurun_out/ab_tscan3.txt
for wl in c5_n511_N1024 c4 c5_n511_N256 c5_n127_N1024; do
  echo "$wl scan $(timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time 2>&1 | tail -1)" >> gpurun_out/ab_tscan3.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tscan" -c 1 -o gpurun_out/prof_tscan -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_tscan.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_tscan.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
