#!/bin/bash
# Round-2 GPU check: smoke, GPU tests, default bench, format sweep, N=2 same-GPU plumbing.
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/r02_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/r02_smoke.log
timeout 600 python bench.py > $OUT/r02_bench.json 2> $OUT/r02_bench.err; echo "bench rc=$?" >> $OUT/r02_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/r02_gpu_tests.log 2>&1; echo "tests rc=$?" >> $OUT/r02_gpu_tests.log
timeout 600 python bench.py --steps 40 --formats 3,0:5,2:4,3:5,6:5,10 --no-cpu-baseline --no-peer-sim > $OUT/r02_bench_formats.json 2> $OUT/r02_bench_formats.err
APS_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $OUT/r02_bench_n2_plumbing.json 2> $OUT/r02_bench_n2_plumbing.err
echo done
