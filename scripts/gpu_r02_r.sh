#!/bin/bash
# k_trivar v3 (tabulated upper tree): parity, timing vs old, phase trace, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_variable or price or c3 or singular or P1 or stage or tv" > gpurun_out/pytest_tv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tv.log
timeout 600 python -m pytest tests/test_shard_gpu.py -q -p no:cacheprovider >> gpurun_out/pytest_tv.log 2>&1; echo "pytest shard exit $?" >> gpurun_out/pytest_tv.log
rm -f gpurun_out/ab_tv.txt
for rep in 1 2; do
  for dbg in 0 512; do
    echo "debug=$dbg $(timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time --debug $dbg 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
  done
done
timeout 120 python scripts/prof_ops.py --workload c3 --op gmres --reps 5 --time > gpurun_out/c3_gmres.txt 2>&1
CNPINT_LIB=paper_2401_16113_b200/libcnpint_trace.so timeout 120 python scripts/trivar_trace.py --workload c3 > gpurun_out/trv_trace.txt 2>&1
bash scripts/gpu_ncu_env.sh c3 "k_trivar<8, 128, true, false>" tv3_c3 X=1
echo done
