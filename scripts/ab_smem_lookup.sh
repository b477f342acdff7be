#!/bin/bash
# Walker A/B: the fast path's shared-memory code lookup (random (top, mid) indices,
# ~3 bank-conflict ways per warp access) vs a probe build that reads one real code per thread and
# chunk and derives the other lanes' codes in registers (wrong results, the same spread of leaf-index
# gathers): how much of the walk the SMEM lookup and its conflicts cost.  Serial C5 step, 10 steps.
# Variant: scripts/build_variant.sh fakecodes -DPV_PROBE_FAKE_CODES
mkdir -p gpurun_out
for v in default fakecodes; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_fakecodes.so; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms 0 \
    > gpurun_out/sm_$v.json 2> gpurun_out/sm_$v.err
  python - "$v" gpurun_out/sm_$v.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>10}: walk {d['translate_ms_per_step']:.4f} ms/step = {d['value'] / 1e9:.1f} G lanes/s")
PY
  timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
    --clock-control none -k regex:"translate_kernel" -c 1 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    --no-e2e --no-parity --split-sms 0 2>/dev/null | grep -E "bank|wavefronts|xbar|duration" | cut -d, -f13- | sed "s/^/  $v ncu: /"
done
