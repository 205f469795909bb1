#!/bin/bash
# A/B the fused p=1 schedules (wavefront vs barrier) in one box session: bash scripts/sched.sh [rounds]
for r in $(seq ${1:-2}); do
  for S in wave barrier; do
    APS_FUSED_SCHEDULE=$S python bench.py --steps 300 --warmup 5 --phase-steps 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$S', round(d['ms_per_step']*1e3,2), 'us', d['value'], 'GB/s')"
  done
done
