#!/bin/bash
# C2: windows per FIFO speculation run (PV_FIFO_RUN 8 default vs 4 / 16).
# Variants: scripts/build_variant.sh fiforun16 -DPV_FIFO_RUN=16; scripts/build_variant.sh fiforun4 -DPV_FIFO_RUN=4
for v in default fiforun4 fiforun16; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
  timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fr_$v.json 2> gpurun_out/fr_$v.err
  python - "$v" gpurun_out/fr_$v.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>10}: {d['ms_per_step']:.3f} ms/step, plan+fifo {d['plan_fifo_ms_per_step']:.3f} ms")
PY
done
