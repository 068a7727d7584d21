#!/bin/bash
# full GPU suite, headline bench + launch list, per-workload op times (after the PDL trigger change)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
bash scripts/gpu_bench.sh
rm -f gpurun_out/times.jsonl
for w in c2 c3 c4 c5_n511_N1024; do
  timeout 300 python scripts/prof_ops.py --workload $w --op all --reps 5 --time >> gpurun_out/times.jsonl 2>> gpurun_out/times.err
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
echo done
