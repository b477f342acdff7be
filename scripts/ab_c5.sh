#!/bin/bash
# A/B the C5 walker over library variants in scripts/variants/ (1 GPU).
orig=$(mktemp); cp paper_1304_3771_b200/libpv.so $orig
for v in scripts/variants/*.so; do
  cp $v paper_1304_3771_b200/libpv.so
  for rep in 1 2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'translate_ms', round(d['translate_ms_per_step'],4), 'exec_ms', round(d['copy']['exec_ms_per_step'],4), 'sol_frac', round(d['roofline_walk']['gather_sol']['frac'],3))"
  done
done
cp $orig paper_1304_3771_b200/libpv.so
