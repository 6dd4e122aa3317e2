#!/bin/bash
cd "$(dirname "$0")/.."
for l in ${LIBS}; do
  for mode in adaptive global; do
    out=$(NH_LIB=$l timeout 300 python bench.py --steps ${STEPS:-200} --warmup 3 --cpu-steps 0 --no-e2e --mode $mode 2>&1 | tail -1)
    echo "$l $mode: $(echo "$out" | python -c "import sys,json
try:
  d=json.loads(sys.stdin.read()); print('%.3f G' % (d['value']/1e9), d['config']['status_ok'])
except Exception as e: print('FAILED')")"
  done
done
