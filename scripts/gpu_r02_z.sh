#!/bin/bash
# headline-only ncu launch list + ncu --set full of the headline kernels and of c3's K3 (after the r02 changes)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-table > gpurun_out/bench_nt.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_headline.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-table > gpurun_out/ncu_launch_h.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch_h.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dst4|k_dst5|k_tpass2" -c 3 -o gpurun_out/prof_c5h -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_c5h.log 2>&1
echo "ncu c5h exit $?" >> gpurun_out/ncu_c5h.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_matvec2d" -c 2 -o gpurun_out/prof_c5g -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op gmres --reps 1 > gpurun_out/ncu_c5g.log 2>&1
echo "ncu c5g exit $?" >> gpurun_out/ncu_c5g.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_trivar" --launch-skip 1 -c 1 -o gpurun_out/prof_c3k3 -f \
    python scripts/prof_ops.py --workload c3 --op pinv --reps 2 > gpurun_out/ncu_c3k3.log 2>&1
echo done
