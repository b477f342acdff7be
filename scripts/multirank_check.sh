#!/bin/bash
# Robustness of the N > 1 bench path at 4 and 8 ranks sharing one GPU (gloo; scaled C5 world):
# sharding, residency, split steps, peer result return, gather, the shared-buffer e2e.
mkdir -p gpurun_out
for n in 4 8; do
  PV_BENCH_SHARED_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 2 --warmup 3 --scale 8 \
    --gather --no-cpu-baseline > gpurun_out/mr_$n.json 2> gpurun_out/mr_$n.err
  echo "N=$n rc=$?"
  python - gpurun_out/mr_$n.json <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1])
print(" lines", len(lines), "n_gpus", d["n_gpus"], "parity", d["parity"]["ok"], "results_to_rank0",
      (d["results_to_rank0"] or {}).get("verified") if isinstance(d["results_to_rank0"], dict) else d["results_to_rank0"],
      "gather", d["gather_to_rank0"]["complete"], "e2e verified", d["e2e"]["gather_to_rank0"]["verified"],
      "step", d["step"]["mode"])
PY
  tail -3 gpurun_out/mr_$n.err
done
