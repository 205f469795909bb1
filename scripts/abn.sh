#!/bin/bash
# A/B/... the N=1 bench step of several libaps builds, interleaved: bash scripts/abn.sh rounds lib1 lib2 ...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    APS_LIB=$L python bench.py --steps 300 --warmup 5 --phase-steps 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L'.split('/')[-1], round(d['ms_per_step']*1e3,2), 'us', d['value'], 'GB/s')"
  done
done
