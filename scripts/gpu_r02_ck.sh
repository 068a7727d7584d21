#!/bin/bash
# after the adaptive 2D matvec chunk: parity of the touched paths, then the bench without the CPU baseline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_shard_gpu.py -q -p no:cacheprovider -x -k "matvec or apply_A or gmres or host_entry or shard" > gpurun_out/pytest_mvs.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mvs.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench exit $?" >> gpurun_out/bench_q.err
