#!/bin/bash
OUT=gpurun_out
T=${1:-r02m}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_mixed.py tests/test_gpu_graph.py tests/test_gpu_census.py tests/test_gpu_sr.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2 3; do timeout 300 python bench.py --steps 60 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'], d['flushed']['us'])"; done > $OUT/${T}_phases.txt 2>&1
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL --kernel-name-base demangled -k regex:'CAOnly' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3 > $OUT/ncu_absmax_$T.log 2>&1
ncu -i $OUT/prof_${T}_absmax.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_absmax_raw.csv 2>&1
echo done
