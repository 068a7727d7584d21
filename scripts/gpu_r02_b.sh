#!/bin/bash
# k_dst2 bring-up: orthogonality debug, the DST parity tests, A/B timings old (debug 256) vs new
mkdir -p gpurun_out
timeout 300 python scripts/dbg_orth.py > gpurun_out/dbg_orth.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dst or negative or pinv_small or timepass" \
   > gpurun_out/pytest_dst.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dst.log
rm -f gpurun_out/ab_dst2.jsonl
for wl in c4 c5_n127_N1024 c5_n255_N1024 c5_n511_N1024; do
  for dbg in 0 256; do
    timeout 300 python scripts/prof_ops.py --workload $wl --op pinv --reps 5 --time --debug $dbg >> gpurun_out/ab_dst2.jsonl 2>> gpurun_out/ab_dst2.err
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dst2" -c 2 -o gpurun_out/prof_dst2_c5 -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_dst2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_dst2.log
