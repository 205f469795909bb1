#!/bin/bash
# sweep one environment variable over values for the N=1 bench step, interleaved:
#   bash scripts/envsweep.sh VAR "v1 v2 ..." [rounds]
for r in $(seq ${3:-2}); do
  for V in $2; do
    env $1=$V python bench.py --steps 300 --warmup 5 --phase-steps 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1=$V', round(d['ms_per_step']*1e3,2), 'us', d['value'], 'GB/s')"
  done
done
