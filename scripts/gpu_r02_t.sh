#!/bin/bash
# k_trivar: α'/γ' in shared memory (APS, 4 CTAs/SM) vs registers (noaps build) vs first generation (debug 512)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "k3_variable or price or c3 or singular or P1 or stage or tv" > gpurun_out/pytest_tv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tv.log
rm -f gpurun_out/ab_tv.txt
for rep in 1 2; do
  echo "aps $(timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
  echo "noaps $(CNPINT_LIB=paper_2401_16113_b200/libcnpint_noaps.so timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
  echo "gen1 $(timeout 120 python scripts/prof_ops.py --workload c3 --op pinv --reps 10 --time --debug 512 2>&1 | tail -1)" >> gpurun_out/ab_tv.txt
done
timeout 120 python scripts/prof_ops.py --workload c3 --op gmres --reps 5 --time > gpurun_out/c3_gmres.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_trivar" --launch-skip 1 -c 1 -o gpurun_out/prof_tv4_c3 -f \
    python scripts/prof_ops.py --workload c3 --op pinv --reps 2 > gpurun_out/ncu_tv4.log 2>&1
echo done
