#!/bin/bash
# Walker CTA shape (512 x 4 lanes default, 256 x 8, 128 x 16 lanes per thread) in the serial and split C5 step.
# Variants: scripts/build_variant.sh tpb256 -DPV_TR1_TPB=256; scripts/build_variant.sh tpb128 -DPV_TR1_TPB=128
mkdir -p gpurun_out
for v in default tpb256 tpb128; do
  for n in 0 64; do
    if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
    timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms $n \
      > gpurun_out/tp_${v}_$n.json 2> gpurun_out/tp_${v}_$n.err
    python - "$v $n" gpurun_out/tp_${v}_$n.json <<'PY'
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
