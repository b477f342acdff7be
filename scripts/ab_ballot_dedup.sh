#!/bin/bash
# North-star walker options A/B: warp-uniform fault path and explicit warp dedup vs the product.
# Variants: scripts/build_variant.sh threadwise -DPV_TR_WARP_BALLOT=0; scripts/build_variant.sh dedup -DPV_TR_DEDUP=1
for v in default threadwise dedup; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
  timeout 600 python scripts/ab_ballot_dedup.py
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --split-sms 0 \
    > gpurun_out/bd_$v.json 2> gpurun_out/bd_$v.err
  python - "$v" gpurun_out/bd_$v.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>22}: C5 random walk {d['translate_ms_per_step']:.4f} ms = {d['value'] / 1e9:.1f} G/s")
PY
done
