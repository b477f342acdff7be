#!/bin/bash
# A/B the C2 ordered apply over library variants in scripts/variants/ (1 GPU).
orig=$(mktemp); cp paper_1304_3771_b200/libpv.so $orig
for v in scripts/variants/*.so; do
  cp $v paper_1304_3771_b200/libpv.so
  timeout 300 python bench.py --workload c2 --steps 5 --warmup 2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'fwd_ms', round(d['forward_ms_per_step'],3), 'plan_fifo_ms', round(d['plan_fifo_ms_per_step'],3), 'apply_ms', round(d['ordered_apply_ms_per_step'],3), 'launch_ms', round(d['roofline']['launch_ms'],3), 'frac', round(d['roofline']['frac'],3))"
done
cp $orig paper_1304_3771_b200/libpv.so
