#!/bin/bash
# Round-2 evidence: walker SOL probe (incl. the packed form), ncu launch lists + full captures, C5 line.
tag=${1:-r02l}
mkdir -p gpurun_out
./scripts/store_probe.bin > gpurun_out/${tag}_store_probe.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/${tag}_store_probe.txt
bash scripts/ncu_round.sh ${tag}
for f in gpurun_out/${tag}_c5_full.ncu-rep gpurun_out/${tag}_c2_full.ncu-rep; do
  [ -f "$f" ] && python profiles/summarize.py full "$f" "${f%.ncu-rep}.md" && echo "summarised $f"
done
[ -f gpurun_out/${tag}_launches_c5.csv ] && python profiles/summarize.py launches gpurun_out/${tag}_launches_c5.csv gpurun_out/${tag}_launches_c5.md
[ -f gpurun_out/${tag}_launches_c2.csv ] && python profiles/summarize.py launches gpurun_out/${tag}_launches_c2.csv gpurun_out/${tag}_launches_c2.md
ls -la gpurun_out/ | grep ${tag}
