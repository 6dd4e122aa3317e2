#!/bin/bash
# A/B over environment settings: ENVS="A=1,B=2 A=3" MODES=... bash tools/ab_env.sh
cd "$(dirname "$0")/.."
for e in ${ENVS}; do
  for mode in ${MODES:-adaptive}; do
    out=$(env $(echo $e | tr ',' ' ') timeout 300 python bench.py --steps ${STEPS:-300} --warmup 3 --cpu-steps 0 --no-e2e --mode $mode 2>&1 | tail -1)
    echo "$e $mode: $(echo "$out" | python -c "import sys,json
try:
  d=json.loads(sys.stdin.read()); s=d['kernel_shares']; print('%.3f G' % (d['value']/1e9), 'ms/step %.3f' % d['ms_per_step'], ' '.join('%s=%.3f' % (k[10:], v['ms_total']/max(1,v['launches'])) for k,v in s.items() if v['launches']>1), d['config']['status_ok'])
except Exception as e: print('FAILED', sys.stdin.read()[-300:])")"
  done
done
