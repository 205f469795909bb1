#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list + one full capture of the
# hot-path kernels of bench.py (N = 1).  Outputs under gpurun_out/.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --phase-steps 3"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py $ARGS > $OUT/bench_under_ncu_$TAG.log 2>&1
# fused p=1 launch (timed step 1) + the three separate stream kernels (phase breakdown)
ncu --set full --clock-control none --import-source on -k 'regex:stream_kernel|fused_p1|absmax|quant_pack|unpack' -s 3 -c 6 \
    -o $OUT/prof_$TAG -f python bench.py $ARGS > $OUT/ncu_full_$TAG.log 2>&1
ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/prof_${TAG}_raw.csv 2>&1
ncu -i $OUT/prof_$TAG.ncu-rep --page details --csv > $OUT/prof_${TAG}_details.csv 2>&1
echo profile done
# peer transport (simulated p = 8, ResNet-50): launch list + full capture of the reduce kernel
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/peer_launches_$TAG.csv \
    python scripts/peer_sim.py 8 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:peer_reduce -s 8 -c 1 \
    -o $OUT/peer_$TAG -f python scripts/peer_sim.py 8 3 > $OUT/ncu_peer_$TAG.log 2>&1
ncu -i $OUT/peer_$TAG.ncu-rep --page raw --csv > $OUT/peer_${TAG}_raw.csv 2>&1
echo peer profile done
