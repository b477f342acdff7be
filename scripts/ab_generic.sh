#!/bin/bash
# 4-level generic walk: lane-by-lane walks (default) vs level-synchronous lanes, and a 3-CTA/SM register cap (level-sync).
# Variants: scripts/build_variant.sh gen_sync -DPV_GEN_LEVELSYNC=1; scripts/build_variant.sh gen_minb3 -DPV_GEN_LEVELSYNC=1 -DPV_GEN_MINB=3
mkdir -p gpurun_out
for v in default gen_sync gen_minb3; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
  for w in c3 c1_4l; do
    if [ $w = c3 ]; then a="--workload c3"; else a="--workload c1 --c1-mode 4l --no-e2e --no-parity"; fi
    timeout 900 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gen_${v}_$w.json 2> gpurun_out/gen_${v}_$w.err
    python - "$v $w" gpurun_out/gen_${v}_$w.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
t = d.get("translate_ms_per_step", d["ms_per_step"])
print(f"{sys.argv[1]:>18}: walk {t * 1e3:.1f} us/step = {d['value'] / 1e9:.1f} G translations/s")
PY
  done
done
