#!/bin/bash
# A/B the separate-call phases (absmax / quant / unpack) of several libaps builds, interleaved:
# bash scripts/ab_absmax.sh rounds lib1 lib2 ...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    APS_LIB=$L python bench.py --steps 20 --warmup 3 --phase-steps 100 --e2e-steps 1 --no-cpu-baseline --no-peer-sim 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['phases']; print('$L'.split('/')[-1], 'absmax', p['absmax_exp']['us'], 'quant', p['quant_pack']['us'], 'unpack', p['unpack_unscale']['us'])"
  done
done
