#!/bin/bash
# staged 2D matvec: which side-vector counts should take it (CNPINT_MVS_MAXNS), with the adaptive chunk
mkdir -p gpurun_out
rm -f gpurun_out/ab_mvs2.txt
for wl in c5_n511_N1024 c4 c5_n255_N1024 c5_n127_N256; do
  for mx in 0 1 2 3; do
    echo "$wl maxns=$mx gmres $(CNPINT_MVS_MAXNS=$mx timeout 300 python scripts/prof_ops.py --workload $wl --op gmres --reps 3 --time 2>&1 | tail -1)" >> gpurun_out/ab_mvs2.txt
    echo "$wl maxns=$mx $(CNPINT_MVS_MAXNS=$mx timeout 300 python scripts/gmres_ab.py --workloads $wl --debugs 0 --reps 5 2>&1 | head -1)" >> gpurun_out/ab_mvs2.txt
  done
  echo "$wl maxns=0 A $(timeout 200 python scripts/prof_ops.py --workload $wl --op A --reps 10 --time 2>&1 | tail -1)" >> gpurun_out/ab_mvs2.txt
done
CNPINT_MVS_MAXNS=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "matvec2d_staged or apply_A or gmres_small or host_entry" > gpurun_out/pytest_mvs.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mvs.log
