#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
T=${1:-r02e}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_mixed.py tests/test_gpu_census.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2; do for L in libaps libaps_absstream; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'])"; done; done > $OUT/${T}_absmax_ab.txt 2>&1
timeout 900 python scripts/ddp_step.py > $OUT/${T}_ddp_step.json 2> $OUT/${T}_ddp_step.err
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:'fused_cw' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py $ARGS --graph 0 > $OUT/ncu_absmax_$T.log 2>&1
echo done
