#!/bin/bash
# TMA bulk copies without (the default) / with the L2 evict-first hint: serial C5 step and the split step.
# Variant: scripts/build_variant.sh evict -DPV_BULK_EVICT_FIRST=1
mkdir -p gpurun_out
for v in default evict; do
  for n in 0 64 72; do
    if [ $v = evict ]; then export PV_LIB=$PWD/scripts/libpv_evict.so; else unset PV_LIB; fi
    timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms $n \
      > gpurun_out/ev_${v}_$n.json 2> gpurun_out/ev_${v}_$n.err
    python - "$v $n" gpurun_out/ev_${v}_$n.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
st = d["step"]
sp = st.get("split") or {}
print(f"{sys.argv[1]:>12}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} walk {d['translate_ms_per_step']:.3f} "
      f"exec {d['copy']['exec_ms_per_step']:.3f} | split walk {sp.get('walk_ms', 0):.3f} exec {sp.get('exec_ms', 0):.3f}")
PY
  done
done
