#!/bin/bash
# Ordered apply: sort (page, u32 chunk index) pairs with the apply gathering descriptors by index (default) vs
# (page, 16 B descriptor) pairs.  Variant: scripts/build_variant.sh ord_desc -DPV_ORD_INDEX=0
mkdir -p gpurun_out
for v in default ord_desc; do
  if [ $v = default ]; then unset PV_LIB; else export PV_LIB=$PWD/scripts/libpv_$v.so; fi
  timeout 900 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/oi_$v.json 2> gpurun_out/oi_$v.err
  python - "$v" gpurun_out/oi_$v.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "failed", e); sys.exit()
k = d.get("kernels", {})
print(f"{sys.argv[1]:>10}: C2 {d['ms_per_step']:.3f} ms/step, apply phase {d['ordered_apply_ms_per_step']:.3f} ms; "
      + ", ".join(f"{n} {v['launch_ms']:.3f}" for n, v in k.items() if n.startswith("ordered")))
PY
done
export PV_LIB=$PWD/scripts/libpv_ord_desc.so
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_configs.py tests/test_gpu_concurrency.py 2>&1 | tail -2
