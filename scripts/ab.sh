#!/bin/bash
# A/B the fused p=1 step of two libaps builds in one box session:
#   bash scripts/ab.sh <libA.so> <libB.so> [rounds]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for L in $A $B; do
    APS_LIB=$L python bench.py --steps 300 --warmup 5 --phase-steps 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L'.split('/')[-1], d['ms_per_step']*1e3, 'us', d['value'], 'GB/s')"
  done
done
