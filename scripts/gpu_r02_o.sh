#!/bin/bash
# K3 variable rows with the tabulated merge tree (MODE_VTAB): parity, A/B vs the generic tree (debug 512), ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_tree or full_c3 or c3_c4 or singular or stage or price or tv or host_entry" > gpurun_out/pytest_vt.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_vt.log
rm -f gpurun_out/ab_vt.jsonl
for dbg in 0 512 0 512; do
  echo "debug $dbg" >> gpurun_out/ab_vt.jsonl
  timeout 300 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time --debug $dbg >> gpurun_out/ab_vt.jsonl 2>> gpurun_out/ab_vt.err
done
timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-table --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tridiag" -c 1 -o gpurun_out/prof_vt -f \
    python scripts/prof_ops.py --workload c3 --op pinv --reps 1 > gpurun_out/ncu_vt.log 2>&1
