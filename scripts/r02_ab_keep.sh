#!/bin/bash
OUT=gpurun_out
T=${1:-r02t}
for r in 1 2; do for L in libaps libaps_k50 libaps_k25; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 40 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'])"; done; done > $OUT/${T}_ab_keep.txt 2>&1
echo done
