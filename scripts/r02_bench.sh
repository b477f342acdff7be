#!/bin/bash
# GPU round trip: optional test files (TESTS="..."), then bench.py with the given args.
tag=$1; shift
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -q -m gpu -p no:cacheprovider -rf > gpurun_out/${tag}_tests.log 2>&1
  echo "tests rc=$?"; tail -n 12 gpurun_out/${tag}_tests.log
fi
timeout 1200 python bench.py "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -n 5 gpurun_out/${tag}_bench.err; tail -c 3000 gpurun_out/${tag}_bench.json
