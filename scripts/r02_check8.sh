#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
T=${1:-r02h}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${T}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${T}_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
FULL="--set full --clock-control none --import-source on --print-units base"
ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv --log-file $OUT/launches_$T.csv python bench.py $ARGS > $OUT/bench_under_ncu_$T.log 2>&1
ncu $FULL --kernel-name-base demangled -k regex:'CAOnly' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py $ARGS > $OUT/ncu_absmax_$T.log 2>&1
ncu $FULL -k regex:'fused_cw' -s 10 -c 1 -o $OUT/prof_${T}_fused -f python bench.py $ARGS > $OUT/ncu_fused_$T.log 2>&1
ncu $FULL -k regex:'fused_cw' -s 10 -c 1 -o $OUT/prof_${T}_fused_e3m0 -f python bench.py $ARGS --format 3,0 > $OUT/ncu_fe3m0_$T.log 2>&1
for r in absmax fused fused_e3m0; do
  ncu -i $OUT/prof_${T}_$r.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_${r}_raw.csv 2>&1
  ncu -i $OUT/prof_${T}_$r.ncu-rep --page source --csv --print-units base > $OUT/prof_${T}_${r}_source.csv 2>&1
done
echo done
