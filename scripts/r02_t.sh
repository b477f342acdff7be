#!/bin/bash
# L2-flushed C1/C3/C4 lines + ncu full captures of the C2 forward / FIFO kernels and the C3 generic walk.
tag=${1:-r02t}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name rc=$?"; tail -n 2 gpurun_out/${tag}_${name}.err; }
run c1 --workload c1 --steps 10 --warmup 3 --no-cpu-baseline
run c3 --workload c3 --steps 10 --warmup 3 --no-cpu-baseline
run c4 --workload c4 --steps 10 --warmup 3 --no-cpu-baseline
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fifo_spec_kernel|frame_pack_kernel|frame_classify_kernel|stamp_kernel|ordered_keys_kernel" -c 5 -o gpurun_out/${tag}_c2b_full \
  python bench.py --workload c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c2b_full.log 2>&1
echo "c2b full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"translate_generic_kernel" -c 1 -o gpurun_out/${tag}_c3_full \
  python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_c3_full.log 2>&1
echo "c3 full rc=$?"
for f in gpurun_out/${tag}_c2b_full.ncu-rep gpurun_out/${tag}_c3_full.ncu-rep; do
  [ -f "$f" ] && python profiles/summarize.py full "$f" "${f%.ncu-rep}.md" && echo "summarised $f"
done
