#!/bin/bash
# A/B the FIFO replay run length over scripts/variants/run*.so (parity tests + C2 bench each), then one ncu capture of fifo_spec_kernel (1 GPU).
orig=$(mktemp); cp paper_1304_3771_b200/libpv.so $orig
for v in scripts/variants/run*.so; do
  cp $v paper_1304_3771_b200/libpv.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fifo or cached or c2" 2>&1 | tail -1
  timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'value', round(d['value']/1e9,3), 'fwd_ms', round(d['forward_ms_per_step'],3), 'plan_fifo_ms', round(d['plan_fifo_ms_per_step'],3), 'apply_ms', round(d['ordered_apply_ms_per_step'],3))"
done
cp $orig paper_1304_3771_b200/libpv.so
[ "${NO_NCU:-0}" = 1 ] || timeout 600 ncu --set full --clock-control none -k regex:"fifo_spec_kernel|fifo_apply_kernel|fifo_verify_kernel" -c 3 -o gpurun_out/fifo_spec python bench.py --workload c2 --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu rc=$?
