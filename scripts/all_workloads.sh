#!/bin/bash
# One bench line per BASELINE workload (c1..c5) and the c2 alpha variants: GMRES time-to-solution and
# iterations, P^-1 applies/s and GB/s, matvec GB/s, per-kernel breakdown (no CPU oracle, one e2e stream).
out=gpurun_out/workloads.jsonl
rm -f $out
for spec in "c1 0.01" "c2 0.1" "c2 0.01" "c2 0.001" "c3 0.01" "c4 0.01" \
            "c5_n127_N256 0.01" "c5_n127_N1024 0.01" "c5_n255_N256 0.01" "c5_n255_N1024 0.01" \
            "c5_n511_N256 0.01" "c5_n511_N1024 0.01"; do
  set -- $spec
  timeout 600 python bench.py --workload $1 --alpha $2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-streams 1 \
      2>> gpurun_out/workloads.err | tail -1 >> $out
done
echo done >> gpurun_out/workloads.err
