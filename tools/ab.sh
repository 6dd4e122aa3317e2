#!/bin/bash
# A/B the step kernel variants on the GPU box.
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-0 1 2 3}; do
  for mode in adaptive global; do
    out=$(NH_STEP_VARIANT=$v timeout 300 python bench.py --steps ${STEPS:-200} --warmup 3 --cpu-steps 0 --no-e2e --mode $mode 2>&1 | tail -1)
    echo "variant $v $mode: $(echo "$out" | python -c "import sys,json
try:
  d=json.loads(sys.stdin.read()); print('%.3f G' % (d['value']/1e9), d['config']['status_ok'])
except Exception as e: print('FAILED')")"
  done
done
