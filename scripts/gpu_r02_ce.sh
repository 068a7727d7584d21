#!/bin/bash
# The headline (c5 n511 N1024) against a full oracle GMRES solve (minutes of CPU), once.
mkdir -p gpurun_out
rm -f gpurun_out/parity_slow.jsonl
CNPINT_SLOW=1 CNPINT_PARITY_LOG=gpurun_out/parity_slow.jsonl timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "largest_vs_oracle" --durations=3 > gpurun_out/pytest_slow.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_slow.log
