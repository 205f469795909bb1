timeout 300 python scripts/steady.py --sets 3 --steps 20 --modes fused > gpurun_out/r02h_first.txt 2>&1; cat gpurun_out/r02h_first.txt
for r in 1 2; do for L in libaps libaps_wave libaps_s4 libaps_lag3 libaps_lag1; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python scripts/steady.py --sets 3 --steps 100 --modes fused 2>&1 | tail -1; done; done > gpurun_out/r02h_steady.txt 2>&1
cat gpurun_out/r02h_steady.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_mixed.py -x -q -k "p1 or graph or mixed" > gpurun_out/r02h_parity.txt 2>&1
tail -15 gpurun_out/r02h_parity.txt
