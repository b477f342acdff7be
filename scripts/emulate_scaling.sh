#!/bin/bash
# Per-rank share of an N-GPU C5 job, run alone on one GPU (PV_BENCH_EMULATE=1: rank 0's guests only, no
# process group), N = 1 2 4 8: what the walker and copier do at each scale (1 GPU).
for n in 1 2 4 8; do
  RANK=0 WORLD_SIZE=$n LOCAL_RANK=0 PV_BENCH_EMULATE=1 timeout 300 python bench.py --gpus $n --steps 10 --warmup 3 \
    --no-e2e --no-cpu-baseline ${@} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('N=$n', 'value(G/s, N x rank-0 share)', round(d['value']/1e9,1), 'translate_ms', round(d['translate_ms_per_step'],4),
      'copy_ms', round(d['copy']['ms_per_step'],4), 'exec_ms', round(d['copy']['exec_ms_per_step'],4),
      'plan_shim_stamp_ms', round(d['copy']['plan_shim_stamp_ms_per_step'],4), 'ms_per_step', round(d['ms_per_step'],4))"
done
