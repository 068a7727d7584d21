#!/bin/bash
# staged 2D matvec (k_matvec2d_s) vs the register kernel (debug 1048576): parity, then timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "matvec2d_staged or apply_A or gmres_small or gmres_c5_vs_oracle or host_entry" > gpurun_out/pytest_mvs.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mvs.log
rm -f gpurun_out/ab_mvs.txt
for wl in c5_n511_N1024 c4 c5_n255_N1024; do
  for dbg in 0 1048576; do
    echo "$wl debug=$dbg A $(timeout 200 python scripts/prof_ops.py --workload $wl --op A --reps 10 --time --debug $dbg 2>&1 | tail -1)" >> gpurun_out/ab_mvs.txt
    echo "$wl debug=$dbg gmres $(timeout 300 python scripts/prof_ops.py --workload $wl --op gmres --reps 3 --time --debug $dbg 2>&1 | tail -1)" >> gpurun_out/ab_mvs.txt
  done
  for tc in 16 64 128; do
    echo "$wl tchunk=$tc A $(CNPINT_MV2_TCHUNK=$tc timeout 200 python scripts/prof_ops.py --workload $wl --op A --reps 10 --time 2>&1 | tail -1)" >> gpurun_out/ab_mvs.txt
  done
  timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0,1048576 --reps 5 >> gpurun_out/ab_mvs.txt 2>&1
done
