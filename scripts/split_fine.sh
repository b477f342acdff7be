#!/bin/bash
# Finer SM partitions (PV_SM_SPLIT_FINE=1: single-SM granularity) around the 64-SM default.
mkdir -p gpurun_out
for n in 64 58 60 62 66 68 70; do
  PV_SM_SPLIT_FINE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity \
    --split-sms $n > gpurun_out/sf_$n.json 2> gpurun_out/sf_$n.err
  python - "$n" gpurun_out/sf_$n.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
st = d["step"]; sp = st.get("split") or {}
print(f"fine {sys.argv[1]:>3}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} sms {sp.get('sms')} walk {sp.get('walk_ms', 0):.3f} exec {sp.get('exec_ms', 0):.3f}")
PY
done
