#!/bin/bash
# C5 step: back to back vs SM split (64) vs co-resident overlap (PV_CONCURRENT walker beside the exec).
mkdir -p gpurun_out
for mode in "--split-sms 0" "--split-sms 64" "--overlap"; do
  tag=$(echo $mode | tr -d ' -')
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity $mode \
    > gpurun_out/ov_$tag.json 2> gpurun_out/ov_$tag.err
  python - "$mode" gpurun_out/ov_$tag.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
st = d["step"]
print(f"{sys.argv[1]:>16}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} mode {st['mode']} "
      f"walk_in_step {st.get('walk_ms_in_overlap')}")
PY
done
