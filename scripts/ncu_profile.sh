#!/bin/bash
# ncu evidence for the bench's kernels (1 GPU).  Usage: bash scripts/ncu_profile.sh tag [scale]
tag=${1:-prof}; scale=${2:-8}
mkdir -p gpurun_out
# launch list of our kernels in a full-size C5 step (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"translate_kernel|plan_kernel|stamp_kernel|exec_kernel" -c 12 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/${tag}_launch_bench.json 2> gpurun_out/${tag}_launch.err
echo "launch list rc=$?"
# full sets of the top kernels on a reduced-size C5 (ncu replays each kernel ~40x)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"translate_kernel|exec_kernel|plan_kernel" -c 3 -o gpurun_out/${tag}_full \
  python bench.py --scale ${scale} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_full.log 2>&1
echo "full rc=$?"
