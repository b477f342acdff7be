#!/bin/bash
# Standard GPU-box round trip: build check, smoke, GPU tests, C5 bench.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag] [extra bench args]
tag=${1:-run}; shift || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" ; tail -n 2 gpurun_out/${tag}_smoke.log
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -n 3 gpurun_out/${tag}_gpu_tests.log
timeout 900 python bench.py "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -n 3 gpurun_out/${tag}_bench.err; cat gpurun_out/${tag}_bench.json
