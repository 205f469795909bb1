#!/bin/bash
# sweep the fused p=1 kernel tuning flags: bash scripts/flags.sh "0 1 2 4 8 15" [rounds]
for r in $(seq ${2:-2}); do
  for F in $1; do
    APS_FUSED_FLAGS=$F python bench.py --steps 300 --warmup 5 --phase-steps 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flags $F', round(d['ms_per_step']*1e3,2), 'us', d['value'], 'GB/s')"
  done
done
