#!/bin/bash
OUT=gpurun_out
T=${1:-r02y2}
APS_LIB=paper_1911_08907_b200/libaps_t2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p1 or every_width" > $OUT/${T}_t2_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_t2_tests.log
for r in 1 2 3; do for L in libaps libaps_t1 libaps_t2; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 100 --phase-steps 5 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['flushed']['us'])"; done; done > $OUT/${T}_ab_tail.txt 2>&1
echo done
