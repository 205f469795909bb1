#!/bin/bash
OUT=gpurun_out
T=${1:-r02p}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_mixed.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2; do for L in libaps libaps_cwabs; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 40 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'])"; done; done > $OUT/${T}_ab_tma.txt 2>&1
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:'absmax_tma' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3 > $OUT/ncu_absmax_$T.log 2>&1
ncu -i $OUT/prof_${T}_absmax.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_absmax_raw.csv 2>&1
echo done
