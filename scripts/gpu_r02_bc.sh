#!/bin/bash
# k_tpass2: GEN 2 (table divide) vs GEN 3 (+ cp.async prefetch, CNPINT_TPASS2_PF=1) vs GEN 1 (debug 262144); parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "timepass" > gpurun_out/pytest_tp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tp.log
rm -f gpurun_out/ab_tp.txt
for rep in 1 2; do
  for wl in c5_n511_N1024 c5_n511_N256 c4; do
    for v in "0 0" "262144 0" "0 1"; do
      set -- $v
      echo "$wl dbg=$1 pf=$2 $(CNPINT_TPASS2_PF=$2 timeout 200 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $1 2>&1 | tail -1 | cut -c1-140)" >> gpurun_out/ab_tp.txt
    done
  done
done
echo done
