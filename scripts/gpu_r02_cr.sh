#!/bin/bash
# derived-norm probe of the last Arnoldi step (2D): parity, then timing against debug 2097152 (probe off)
mkdir -p gpurun_out
rm -f gpurun_out/parity_probe.jsonl gpurun_out/ab_probe.txt
CNPINT_PARITY_LOG=gpurun_out/parity_probe.jsonl timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "derived_norm or gmres_small or gmres_restart or gmres_c5_vs_oracle or orthogonality or gmres_c4 or host_entry or gram" > gpurun_out/pytest_probe.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_probe.log
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 2097152,0 --reps 5 >> gpurun_out/ab_probe.txt 2>&1
done
