#!/bin/bash
# shard tests + ESINGULAR + DMMA-vs-FFT + ncu of the headline's dominant kernels + launch list
mkdir -p gpurun_out
CNPINT_PARITY_LOG=gpurun_out/parity_shard.jsonl timeout 1800 python -m pytest tests/test_shard_gpu.py tests/test_gpu_parity.py -q -p no:cacheprovider \
   -k "shard or singular" > gpurun_out/pytest_shard.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_shard.log
timeout 600 python scripts/dmma_dst_ab.py > gpurun_out/dmma_dst_ab.json 2> gpurun_out/dmma_dst_ab.err
timeout 600 ncu --set full --clock-control none -k regex:"gemm|Gemm" -c 1 -o gpurun_out/prof_dgemm -f \
    python scripts/dmma_dst_ab.py > gpurun_out/ncu_dgemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dst|k_tfft" -c 3 -o gpurun_out/prof_c5big -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op pinv --reps 1 > gpurun_out/ncu_c5big.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c5big.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-table --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_launch.log
