#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
T=${1:-r02c}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_mixed.py tests/test_gpu_ddp.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 --no-peer-sim > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
timeout 900 python scripts/ddp_step.py > $OUT/${T}_ddp_step.json 2> $OUT/${T}_ddp_step.err
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:'absmax_stream' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py $ARGS > $OUT/ncu_absmax_$T.log 2>&1
ncu -i $OUT/prof_${T}_absmax.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_absmax_raw.csv 2>&1
ncu -i $OUT/prof_${T}_absmax.ncu-rep --page source --csv --print-units base > $OUT/prof_${T}_absmax_source.csv 2>&1
echo done
