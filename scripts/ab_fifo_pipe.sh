#!/bin/bash
# FIFO-10 speculation kernel: software-pipelined window loads at 3 CTAs/SM (default, 80 registers) vs loads at
# each window (PV_FIFO_PIPE=0, 4 CTAs/SM, 61 registers) vs pipelined at 4 CTAs/SM (64 registers, spills).
# Variants: scripts/build_variant.sh fifo_nopipe -DPV_FIFO_PIPE=0; scripts/build_variant.sh fifo_pipe4 -DPV_FIFO_SPEC_MINB=4
mkdir -p gpurun_out
for v in default fifo_nopipe fifo_pipe4; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
  timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fp_$v.json 2> gpurun_out/fp_$v.err
  python - "$v" gpurun_out/fp_$v.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
k = d.get("kernels", {})
print(f"{sys.argv[1]:>12}: C2 {d['ms_per_step']:.3f} ms/step, plan+fifo {d['plan_fifo_ms_per_step']:.3f} ms, "
      f"fifo_spec {k.get('fifo_spec', {}).get('launch_ms', 0):.3f} ms/launch; "
      + ", ".join(f"{n} {v['launch_ms']:.3f}" for n, v in k.items()))
PY
done
