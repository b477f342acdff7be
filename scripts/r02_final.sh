#!/bin/bash
# Round-2 refresh: every bench line, then the whole GPU suite.
tag=${1:-r02m}
bash scripts/r02_benches.sh ${tag}
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/${tag}_all.log 2>&1
echo "all rc=$?"; tail -n 6 gpurun_out/${tag}_all.log
