#!/bin/bash
OUT=gpurun_out
T=${1:-r02x}
for r in 1 2; do for L in libaps libaps_b4m4 libaps_b4m3; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python scripts/peer_sim.py 8 12 2>&1 | tail -1; done; done > $OUT/${T}_peer_batch_ab.txt 2>&1
echo done
