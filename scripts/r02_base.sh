#!/bin/bash
# Round-2 re-entry check: the whole GPU suite at HEAD, then per-call latency.
tag=${1:-r02c}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -n 6 gpurun_out/${tag}_gpu_tests.log
timeout 600 python scripts/percall_latency.py > gpurun_out/${tag}_percall.json 2> gpurun_out/${tag}_percall.err
echo "percall rc=$?"; tail -c 3000 gpurun_out/${tag}_percall.json; tail -n 5 gpurun_out/${tag}_percall.err
