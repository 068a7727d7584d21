#!/bin/bash
# full GPU suite after the ESINGULAR / orthogonality fixes + A/B of the 2D sine-pass kernels
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/ab_dstreg.jsonl
for wl in c4 c5_n127_N1024 c5_n255_N1024 c5_n511_N1024; do
  for dbg in 0 1024 256; do
    echo "debug $dbg" >> gpurun_out/ab_dstreg.jsonl
    timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg >> gpurun_out/ab_dstreg.jsonl 2>> gpurun_out/ab_dstreg.err
  done
done
