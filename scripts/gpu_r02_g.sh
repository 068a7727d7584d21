#!/bin/bash
# full GPU suite + bench (pipelined e2e) + ncu of the cuBLAS DGEMM (dense DST on DMMA)
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none -k regex:"Kernel2" -c 1 -o gpurun_out/prof_dgemm -f \
    python scripts/dmma_dst_ab.py > gpurun_out/ncu_dgemm.log 2>&1
