#!/bin/bash
# ncu evidence for every bench line (1 GPU).  Usage: bash scripts/ncu_round.sh tag
# 1. launch lists (gpu__time_duration per launch, cold-cache, serialised) of a C5 and a C2 step;
# 2. one `--set full` capture of each dominant kernel at full size (DRAM bytes -> roofline traffic).
tag=${1:-prof}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^(translate|stage|plan|stamp|exec|shim)" -c 16 --csv \
  --log-file gpurun_out/${tag}_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --split-sms 0 \
  > gpurun_out/${tag}_launch_c5.json 2> gpurun_out/${tag}_launch_c5.err
echo "c5 launch list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"pv::|CUB_" -c 60 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --workload c2 --steps 2 --warmup 1 \
  > gpurun_out/${tag}_launch_c2.json 2> gpurun_out/${tag}_launch_c2.err
echo "c2 launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"translate_kernel|exec_bulk_kernel|exec_kernel" -c 2 -o gpurun_out/${tag}_c5_full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --split-sms 0 > gpurun_out/${tag}_c5_full.log 2>&1
echo "c5 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"ordered_apply_kernel|fifo_spec_kernel|plan_kernel|Onesweep" -c 5 -o gpurun_out/${tag}_c2_full \
  python bench.py --workload c2 --steps 1 --warmup 1 > gpurun_out/${tag}_c2_full.log 2>&1
echo "c2 full rc=$?"
