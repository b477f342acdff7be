#!/bin/bash
# Walker evidence (1 GPU): C5 / C1 translate times, then one ncu --set full capture of the C5 translate
# kernel (stage pre-pass included).
for w in c5 c1 c4; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$w', 'translate_ms', round(d['translate_ms_per_step'],4), 'G/s', round(d['value']/1e9,1), 'ms_per_step', round(d['ms_per_step'],4))"
done
[ "${NO_NCU:-0}" = 1 ] || timeout 900 ncu --set full --clock-control none --import-source on -k regex:"translate_kernel|stage_table" -c 2 \
  -o gpurun_out/walk_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
