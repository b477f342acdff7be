#!/bin/bash
# Walker A/B (1 GPU): C5 translate time for the CTA-shape tuning hook, then one ncu --set full capture of
# the C5 translate kernel (stage pre-pass included).
for tpb in 512 1024 128; do
  PV_TRANSLATE_TPB=$tpb timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tpb $tpb', 'translate_ms', round(d['translate_ms_per_step'],4), 'G/s', round(d['value']/1e9,1))"
done
[ "${NO_NCU:-0}" = 1 ] || timeout 900 ncu --set full --clock-control none --import-source on -k regex:"translate_kernel|stage_table" -c 2 \
  -o gpurun_out/walk_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
