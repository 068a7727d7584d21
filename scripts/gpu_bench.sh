#!/bin/bash
# full bench (default config) + ncu launch list of the same command
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_launch.log
