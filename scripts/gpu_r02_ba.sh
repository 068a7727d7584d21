#!/bin/bash
# round 2 re-entry (session 5): smoke, the GPU suite (parity log), the headline bench at HEAD.
mkdir -p gpurun_out
( nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv ) > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
