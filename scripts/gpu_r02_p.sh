#!/bin/bash
# K3 variable rows, dense-tree kernel: parity, A/B (default MINB 4 / tv3 / tv5 builds / debug 512 old kernel), ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_variable or price or c3 or singular or P1" > gpurun_out/pytest_tv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tv.log
rm -f gpurun_out/ab_tv.txt
for rep in 1 2; do
  for lib in "" tv3 tv5; do
    for dbg in 0 512; do
      [ -n "$lib" ] && [ $dbg = 512 ] && continue
      L=""; [ -n "$lib" ] && L="CNPINT_LIB=paper_2401_16113_b200/libcnpint_$lib.so"
      echo "lib=${lib:-default} debug=$dbg $(env $L timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time --debug $dbg 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
    done
  done
done
bash scripts/gpu_ncu_env.sh c3 "k_trivar" tv_c3 X=1
CNPINT_LIB=paper_2401_16113_b200/libcnpint_tv3.so bash scripts/gpu_ncu_env.sh c3 "k_trivar" tv3_c3 X=1
echo done
