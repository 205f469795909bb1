#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list of bench.py (N = 1) and one full capture
# of each hot-path kernel (base units: --print-units base).  Outputs under gpurun_out/.
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py $ARGS > $OUT/bench_under_ncu_$TAG.log 2>&1
FULL="--set full --clock-control none --import-source on --print-units base"
# the fused N = 1 launch (a launch of the steady-state loop), then the separate-call kernels (N > 1 path)
ncu $FULL -k regex:fused_cw -s 10 -c 1 -o $OUT/prof_${TAG}_fused -f python bench.py $ARGS > $OUT/ncu_fused_$TAG.log 2>&1
ncu $FULL -k regex:'quant_pack|unpack_unscale' -s 6 -c 2 -o $OUT/prof_${TAG}_calls -f python bench.py $ARGS > $OUT/ncu_calls_$TAG.log 2>&1
ncu $FULL --kernel-name-base demangled -k regex:'CAOnly' -s 2 -c 1 -o $OUT/prof_${TAG}_absmax -f python bench.py $ARGS > $OUT/ncu_absmax_$TAG.log 2>&1
for r in fused calls absmax; do
  ncu -i $OUT/prof_${TAG}_$r.ncu-rep --print-units base --page raw --csv > $OUT/prof_${TAG}_${r}_raw.csv 2>&1
  ncu -i $OUT/prof_${TAG}_$r.ncu-rep --print-units base --page details --csv > $OUT/prof_${TAG}_${r}_details.csv 2>&1
  ncu -i $OUT/prof_${TAG}_$r.ncu-rep --page source --csv --print-units base > $OUT/prof_${TAG}_${r}_source.csv 2>&1
done
echo profile done
# peer transport (simulated p = 8, ResNet-50): launch list + full capture of the reduce kernel
ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv --log-file $OUT/peer_launches_$TAG.csv \
    python scripts/peer_sim.py 8 2 > /dev/null 2>&1
ncu $FULL -k regex:peer_reduce -s 8 -c 1 -o $OUT/peer_$TAG -f python scripts/peer_sim.py 8 3 > $OUT/ncu_peer_$TAG.log 2>&1
ncu -i $OUT/peer_$TAG.ncu-rep --print-units base --page raw --csv > $OUT/peer_${TAG}_raw.csv 2>&1
echo peer profile done
