#!/bin/bash
# A/B the separate-call phase kernels of two builds: bash scripts/ab_phases.sh libA libB [rounds]
for r in $(seq ${3:-2}); do
  for L in $1 $2; do
    APS_LIB=$L python bench.py --steps 40 --warmup 5 --phase-steps 100 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['phases']; print('$L'.split('/')[-1], ' '.join(f'{k}={v[\"us\"]}' for k,v in p.items()))"
  done
done
