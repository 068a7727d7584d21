#!/bin/bash
# orthogonality test + compute-sanitizer (memcheck, racecheck, synccheck) on the kernel families
mkdir -p gpurun_out
timeout 300 python scripts/dbg_orth.py > gpurun_out/dbg_orth.log 2>&1
CNPINT_PARITY_LOG=gpurun_out/parity_orth.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "orthogonality or singular or binding or peak" \
   > gpurun_out/pytest_orth.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_orth.log
rm -f gpurun_out/sanitize.txt
for case in c1 fourstep var cluster2d reg2d dst2 classic; do
  for tool in memcheck racecheck synccheck; do
    echo "=== $case $tool" >> gpurun_out/sanitize.txt
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py --case $case >> gpurun_out/sanitize.txt 2>&1
    echo "exit $?" >> gpurun_out/sanitize.txt
  done
done
