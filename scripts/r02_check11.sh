#!/bin/bash
OUT=gpurun_out
T=${1:-r02k}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_mixed.py tests/test_gpu_peer.py tests/test_gpu_peer_ipc.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2; do for L in libaps libaps_fsc; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python scripts/peer_sim.py 8 12 2>&1 | tail -1; done; done > $OUT/${T}_peer_fence_ab.txt 2>&1
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 --no-cpu-baseline > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
FULL="--set full --clock-control none --import-source on --print-units base"
ncu $FULL -k regex:peer_reduce -s 8 -c 1 -o $OUT/peer_$T -f python scripts/peer_sim.py 8 3 > $OUT/ncu_peer_$T.log 2>&1
ncu -i $OUT/peer_$T.ncu-rep --print-units base --page raw --csv > $OUT/peer_${T}_raw.csv 2>&1
echo done
