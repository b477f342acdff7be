#!/bin/bash
# GPU round trip: selected test files (args), then optionally the whole GPU suite (ALL=1).
tag=$1; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest "$@" -q -m gpu -p no:cacheprovider -x -rf > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -n 30 gpurun_out/${tag}_tests.log
if [ "$ALL" = "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/${tag}_all.log 2>&1
  echo "all rc=$?"; tail -n 8 gpurun_out/${tag}_all.log
fi
