#!/bin/bash
# Run one reference test (file + -k expression) through the drop-in, printing its output.
# usage: scripts/refsuite_one.sh test_acceptance.py c06 [extra env assignments via env]
R=$(cd "$(dirname "$0")/.." && pwd)
export PYTHONPATH="$R/baseline/_ref:$R:$R/tests:$PYTHONPATH" PYTHONDONTWRITEBYTECODE=1
d=$(mktemp -d)
cd "$d" && python -m pytest "$R/baseline/_ref/devfsim_tests/$1" -k "$2" -q -s -p refsuite_plugin -p no:cacheprovider \
  -o addopts= --rootdir "$R/baseline/_ref/devfsim_tests" 2>&1 | grep -E "ACCEPTANCE|passed|failed|Error" | head -20
