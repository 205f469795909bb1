#!/bin/bash
OUT=gpurun_out
T=${1:-r02v}
for r in 1 2; do for L in libaps libaps_s2 libaps_cw2; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 100 --phase-steps 10 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['flushed']['us'], {k:v['us'] for k,v in d['phases'].items()})"; done; done > $OUT/${T}_ab_cw.txt 2>&1
echo done
