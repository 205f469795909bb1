#!/bin/bash
OUT=gpurun_out
T=${1:-r02anc}
APS_LIB=paper_1911_08907_b200/libaps_anc.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p1_resnet50_full or calls" > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2 3; do for L in libaps libaps_anc; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 100 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:v['us'] for k,v in d['phases'].items()})"; done; done > $OUT/${T}_ab.txt 2>&1
echo done
