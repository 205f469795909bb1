for r in 1 2; do for L in libaps_wave libaps_nowait libaps_noa libaps_wave3; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so python scripts/steady.py --sets 3 --steps 100 --modes fused 2>&1 | tail -1; done; done > gpurun_out/r02f_steady.txt 2>&1
cat gpurun_out/r02f_steady.txt
