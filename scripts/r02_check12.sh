#!/bin/bash
OUT=gpurun_out
T=${1:-r02l}
timeout 900 python bench.py --config c5 --steps 30 --no-cpu-baseline > $OUT/${T}_c5.json 2> $OUT/${T}_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${T}_reference.json 2> $OUT/${T}_reference.err
timeout 900 python bench.py --config c3 --format 4,3 --steps 20 --no-cpu-baseline --no-peer-sim > $OUT/${T}_c3.json 2> $OUT/${T}_c3.err
# steady-state DRAM bytes per sync: application replay keeps the caches as the program leaves them
ncu --replay-mode application --cache-control none --clock-control none --print-units base \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:fused_cw -s 12 -c 3 --csv --log-file $OUT/${T}_fused_steady_dram.csv \
    python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3 > $OUT/${T}_ncu_app.log 2>&1
echo done
