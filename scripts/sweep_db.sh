#!/bin/bash
rm -f gpurun_out/sweepdb.jsonl
CNPINT_TFFT_DB=1 timeout 600 python -m pytest tests -m gpu -x -q -k "pinv or stage" > gpurun_out/pytest_db.log 2>&1; echo "exit $?" >> gpurun_out/pytest_db.log
for w in c2 c4 c3; do
for C in 1 2 4 8; do
for DB in 0 1; do
  echo "{\"C\": $C, \"DB\": $DB, \"w\": \"$w\"}" >> gpurun_out/sweepdb.jsonl
  CNPINT_TFFT_DB=$DB CNPINT_TFFT_C=$C timeout 120 python scripts/prof_ops.py --workload $w --op pinv --reps 5 --time >> gpurun_out/sweepdb.jsonl 2>>gpurun_out/sweepdb.err
done
done
done
