#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list + one full capture of the
# three N=1 hot-path kernels of bench.py.  Outputs under gpurun_out/.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_under_ncu_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:absmax|quant_pack|unpack_unscale' -s 9 -c 3 \
    -o $OUT/prof_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_full_$TAG.log 2>&1
ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/prof_${TAG}_raw.csv 2>&1
ncu -i $OUT/prof_$TAG.ncu-rep --page details --csv > $OUT/prof_${TAG}_details.csv 2>&1
echo profile done
