#!/bin/bash
# Copy exec A/B on the C5 bench (1 GPU): TMA bulk exec (default for co-aligned batches) vs the LSU exec.
for v in 0 1 0 1; do
  PV_EXEC_LSU=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['copy']
print('PV_EXEC_LSU=$v', 'exec_ms', round(c['exec_ms_per_step'],4), 'exec GB/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],4), 'copy GB/s', round(c['value']))"
done
