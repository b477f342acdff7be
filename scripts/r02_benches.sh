#!/bin/bash
# Round-2 bench sweep: C5 (default line), C1 (shadow, tdp, 4-level), C2, C4, C3.
tag=${1:-r02}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name rc=$?"; tail -n 2 gpurun_out/${tag}_${name}.err; }
run c5 --steps 10 --warmup 3
run c1 --workload c1 --steps 10 --warmup 3
run c1tdp --workload c1 --c1-mode tdp --steps 10 --warmup 3 --no-cpu-baseline
run c1_4l --workload c1 --c1-mode 4l --steps 10 --warmup 3
run c2 --workload c2 --steps 10 --warmup 3
run c4 --workload c4 --steps 10 --warmup 3
run c3 --workload c3 --steps 10 --warmup 3
run ref --impl reference --steps 3 --warmup 1
