#!/bin/bash
# The 64-SM split with and without single-SM granularity, alternated three times.
mkdir -p gpurun_out
for r in 1 2 3; do
  for f in 0 1; do
    PV_SM_SPLIT_FINE=$f timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity \
      --split-sms 64 > gpurun_out/sfab_$f.json 2> gpurun_out/sfab_$f.err
    python - "$f" gpurun_out/sfab_$f.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
st = d["step"]; sp = st.get("split") or {}
print(f"fine={sys.argv[1]}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} walk {sp.get('walk_ms', 0):.3f} exec {sp.get('exec_ms', 0):.3f}")
PY
  done
done
