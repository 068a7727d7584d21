#!/bin/bash
# Round-2 closing run: whole GPU suite with the parity log, smoke, the bench, the headline-only ncu launch list,
# ncu --set full of the staged 2D matvec, per-kernel timings of every workload.
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl gpurun_out/times.jsonl
CNPINT_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-table > gpurun_out/bench_nt.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_headline.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-table > gpurun_out/ncu_launch_h.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch_h.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_matvec2d_s" -c 1 -o gpurun_out/prof_mvs -f \
    python scripts/prof_ops.py --workload c5_n511_N1024 --op A --reps 1 > gpurun_out/ncu_mvs.log 2>&1
echo "ncu mvs exit $?" >> gpurun_out/ncu_mvs.log
for w in c1 c2 c3 c4 c5_n511_N1024; do
  timeout 300 python scripts/prof_ops.py --workload $w --op all --reps 5 --time >> gpurun_out/times.jsonl 2>> gpurun_out/times.err
done
echo done
