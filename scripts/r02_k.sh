#!/bin/bash
tag=${1:-r02k}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name rc=$?"; tail -n 2 gpurun_out/${tag}_${name}.err; }
run c2 --workload c2 --steps 10 --warmup 3 --no-cpu-baseline
run c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
run c5p --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --packed
timeout 600 python scripts/percall_latency.py > gpurun_out/${tag}_percall.json 2> gpurun_out/${tag}_percall.err; echo "percall rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/${tag}_all.log 2>&1
echo "all rc=$?"; tail -n 6 gpurun_out/${tag}_all.log
