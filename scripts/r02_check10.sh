#!/bin/bash
OUT=gpurun_out
T=${1:-r02j}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_mixed.py tests/test_gpu_ddp.py tests/test_gpu_peer.py -x -q > $OUT/${T}_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_tests.log
for r in 1 2; do for L in libaps libaps_dynfirst; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 60 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'], d['flushed']['us'])"; done; done > $OUT/${T}_ab_static.txt 2>&1
timeout 600 python bench.py --formats 3,0:5,6 --no-cpu-baseline --no-peer-sim --no-parity > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
echo done
