#!/bin/bash
# Walker next-chunk VA prefetch (PV_TR_PREFETCH=1) in the serial and the split C5 step: the split walk is
# latency-bound (its VA loads queue behind the copy's HBM traffic), the serial one port-bound.
# Variant: scripts/build_variant.sh prefetch -DPV_TR_PREFETCH=1
mkdir -p gpurun_out
for v in default prefetch; do
  for n in 0 64; do
    if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
    timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms $n \
      > gpurun_out/pf_${v}_$n.json 2> gpurun_out/pf_${v}_$n.err
    python - "$v $n" gpurun_out/pf_${v}_$n.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
st = d["step"]; sp = st.get("split") or {}
print(f"{sys.argv[1]:>12}: ms/step {d['ms_per_step']:.3f} serial {st['serial_ms']:.3f} walk {d['translate_ms_per_step']:.3f} | split walk {sp.get('walk_ms', 0):.3f} exec {sp.get('exec_ms', 0):.3f}")
PY
  done
done
