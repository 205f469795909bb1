#!/bin/bash
OUT=gpurun_out
T=${1:-r02s}
timeout 1500 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
timeout 600 python bench.py --hybrid --hybrid-last 5,6 --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid56.json 2> $OUT/${T}_hybrid56.err
timeout 600 python bench.py --hybrid --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid32.json 2> $OUT/${T}_hybrid32.err
timeout 600 python bench.py --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_uniform.json 2> $OUT/${T}_uniform.err
echo done
