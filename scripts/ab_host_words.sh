#!/bin/bash
# A/B of the host word pipeline's shape (dataplane._translate_host_words): lanes per chunk x
# chunk buffer sets in flight, on the C5 e2e translate leg (bench.py's default line).
mkdir -p gpurun_out
for v in "8388608 2" "2097152 2" "2097152 4" "4194304 3" "1048576 4" "2097152 6"; do
  set -- $v
  for rep in 1 2; do
    PV_HOST_WORD_CHUNK=$1 PV_HOST_WORD_BUFS=$2 timeout 600 python bench.py --no-parity --no-cpu-baseline \
      --steps 10 --warmup 3 2>/dev/null | tail -n1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('chunk=$1 bufs=$2 rep=$rep', 'e2e %.4g translations/s' % e['value'],
      'translate_ms mean %.3f best %.3f' % (e['translate_ms_per_step']['mean'], e['translate_ms_per_step']['best']))"
  done
done
