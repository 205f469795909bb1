#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
T=${1:-r02d}
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -x -q -k "peer or every_width or c1_and_edges or resnet50_full or sim" > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
timeout 600 python bench.py --steps 60 --no-cpu-baseline > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
for r in 1 2; do for L in libaps libaps_peercvt; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python scripts/peer_sim.py 8 12 2>&1 | tail -1; done; done > $OUT/${T}_peer_ab.txt 2>&1
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 --phase-steps 3"
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:'absmax_stream' -s 2 -c 1 -o $OUT/prof_${T}_absmax -f python bench.py $ARGS > $OUT/ncu_absmax_$T.log 2>&1
ncu $FULL -k regex:'quant_pack|unpack' -s 4 -c 2 -o $OUT/prof_${T}_e3m0 -f python bench.py $ARGS --format 3,0 > $OUT/ncu_e3m0_$T.log 2>&1
ncu $FULL -k regex:'fused_cw' -s 8 -c 1 -o $OUT/prof_${T}_fused_e3m0 -f python bench.py $ARGS --format 3,0 > $OUT/ncu_fe3m0_$T.log 2>&1
ncu $FULL -k regex:peer_reduce -s 8 -c 1 -o $OUT/peer_$T -f python scripts/peer_sim.py 8 3 > $OUT/ncu_peer_$T.log 2>&1
for r in absmax e3m0 fused_e3m0; do
  ncu -i $OUT/prof_${T}_$r.ncu-rep --print-units base --page raw --csv > $OUT/prof_${T}_${r}_raw.csv 2>&1
  ncu -i $OUT/prof_${T}_$r.ncu-rep --page source --csv --print-units base > $OUT/prof_${T}_${r}_source.csv 2>&1
done
ncu -i $OUT/peer_$T.ncu-rep --print-units base --page raw --csv > $OUT/peer_${T}_raw.csv 2>&1
echo done
