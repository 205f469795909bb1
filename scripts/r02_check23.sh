#!/bin/bash
OUT=gpurun_out
T=${1:-r02u}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_graph.py tests/test_gpu_ddp.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2 3; do timeout 300 python bench.py --steps 100 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 4 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'], d['flushed']['us'], d['e2e']['value'])"; done > $OUT/${T}_bench3.txt 2>&1
echo done
