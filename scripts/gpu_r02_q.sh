#!/bin/bash
# k_trivar phase trace (experiment builds) + variable-row parity
mkdir -p gpurun_out
for lib in trace trace4; do
  echo "== $lib" >> gpurun_out/trv_trace.txt
  CNPINT_LIB=paper_2401_16113_b200/libcnpint_$lib.so timeout 120 python scripts/trivar_trace.py --workload c3 >> gpurun_out/trv_trace.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_variable" > gpurun_out/pytest_tv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tv.log
