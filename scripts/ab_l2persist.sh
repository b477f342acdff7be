#!/bin/bash
# C5 split step with the leaf index persisting in L2 for the walk's partition (hit ratio 0 / 0.5 / 1.0).
mkdir -p gpurun_out
for r in 0 0.5 1.0; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --l2-persist $r \
    > gpurun_out/l2p_$r.json 2> gpurun_out/l2p_$r.err
  python - "$r" gpurun_out/l2p_$r.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
st = d["step"]
sp = st.get("split") or {}
print(f"persist {sys.argv[1]:>4}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} split walk {sp.get('walk_ms', 0):.3f} exec {sp.get('exec_ms', 0):.3f} serial walk {d['translate_ms_per_step']:.3f}")
PY
done
tail -3 gpurun_out/l2p_1.0.err
