#!/bin/bash
# A/B of the a1-alone launch: in-flight depth and CTAs per SM (bench phases, flushed, 20 steps)
OUT=gpurun_out
T=${1:-r02i}
for r in 1 2; do for L in libaps libaps_d1 libaps_d2 libaps_c2 libaps_c2d2; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 20 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'])"; done; done > $OUT/${T}_ab_abs.txt 2>&1
echo done
