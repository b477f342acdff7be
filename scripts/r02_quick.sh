#!/bin/bash
# quick round trip: GPU tests (optionally a -k filter) + one bench workload
tag=$1; kexpr=$2; shift 2
mkdir -p gpurun_out
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "$kexpr" > gpurun_out/${tag}_tests.log 2>&1
  echo "tests rc=$?"; tail -n 4 gpurun_out/${tag}_tests.log
fi
if [ $# -gt 0 ]; then
  timeout 900 python bench.py "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
  echo "bench rc=$?"; tail -n 3 gpurun_out/${tag}_bench.err; tail -c 2500 gpurun_out/${tag}_bench.json
fi
