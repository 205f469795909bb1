#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
T=${1:-r02f}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_mixed.py tests/test_gpu_ddp.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 --no-peer-sim --no-cpu-baseline > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
timeout 900 python scripts/ddp_step.py > $OUT/${T}_ddp_step.json 2> $OUT/${T}_ddp_step.err
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:'CAOnly' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py $ARGS > $OUT/ncu_absmax_$T.log 2>&1
ncu $FULL -k regex:'quant_pack|unpack' -s 4 -c 2 -o $OUT/prof_${T}_e3m0 -f python bench.py $ARGS --format 3,0 > $OUT/ncu_e3m0_$T.log 2>&1
ncu $FULL -k regex:'quant_pack|unpack' -s 4 -c 2 -o $OUT/prof_${T}_e5m6 -f python bench.py $ARGS --format 5,6 > $OUT/ncu_e5m6_$T.log 2>&1
for r in absmax e3m0 e5m6; do
  ncu -i $OUT/prof_${T}_$r.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_${r}_raw.csv 2>&1
  ncu -i $OUT/prof_${T}_$r.ncu-rep --page source --csv --print-units base > $OUT/prof_${T}_${r}_source.csv 2>&1
done
echo done
