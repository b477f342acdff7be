#!/bin/bash
# C5 step: phases back to back vs walk and plan+exec on disjoint SM partitions (pv_sm_split).
mkdir -p gpurun_out
tag=${1:-split}
for n in ${SIZES:-0 40 48 56 64}; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms $n \
    > gpurun_out/${tag}_$n.json 2> gpurun_out/${tag}_$n.err
  python - "$n" gpurun_out/${tag}_$n.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
st = d["step"]
print(f"split {sys.argv[1]:>3}: ms/step {d['ms_per_step']:.3f}  serial {st['serial_ms']:.3f}  split {json.dumps(st.get('split'))}")
PY
done
