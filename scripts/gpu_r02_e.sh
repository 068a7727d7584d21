#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/dbg_sing.py > gpurun_out/dbg_sing.log 2>&1
CNPINT_PARITY_LOG=gpurun_out/parity_shard.jsonl timeout 1800 python -m pytest tests/test_shard_gpu.py -q -p no:cacheprovider -x \
   > gpurun_out/pytest_shard.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_shard.log
