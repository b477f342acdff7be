#!/bin/bash
# A/B libpv.so variants in scripts/variants/*.so on one bench workload (1 GPU): each variant runs the
# GPU tests matching $K (if set), then the bench ($W, default c5); the in-tree library is restored after.
W=${W:-c5}
orig=$(mktemp); cp paper_1304_3771_b200/libpv.so $orig
for v in scripts/variants/*.so; do
  cp $v paper_1304_3771_b200/libpv.so
  [ -n "$K" ] && timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "$K" 2>&1 | tail -1
  timeout 300 python bench.py --workload $W $BARGS --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
c = d.get('copy') if isinstance(d.get('copy'), dict) else {}
print('$v', 'value', round(d['value']/1e9,2), 'translate_ms', d.get('translate_ms_per_step'), 'exec_ms', c.get('exec_ms_per_step'),
      'roofline', round(d.get('roofline', {}).get('frac', 0), 4), 'ms_per_step', round(d['ms_per_step'],4))"
done
cp $orig paper_1304_3771_b200/libpv.so
