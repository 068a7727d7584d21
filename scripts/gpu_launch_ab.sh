#!/bin/bash
# ncu launch lists (durations only) of one c2 GMRES solve with debug flags 0 and 128
for d in 0 128; do
  python scripts/prof_ops.py --workload c2 --op gmres --reps 1 --debug $d > gpurun_out/plain_la_$d.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/la_$d.csv python scripts/prof_ops.py --workload c2 --op gmres --reps 1 --debug $d > gpurun_out/ncu_la_$d.log 2>&1
done
