#!/bin/bash
OUT=gpurun_out
T=${1:-r02q}
for r in 1 2; do for L in libaps libaps_c4 libaps_c4d3 libaps_c5; do echo "== $L"; APS_LIB=paper_1911_08907_b200/$L.so timeout 300 python bench.py --steps 40 --phase-steps 30 --no-cpu-baseline --no-parity --no-peer-sim --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v['us'] for k,v in d['phases'].items()}, d['ms_per_step'])"; done; done > $OUT/${T}_ab_abs_occ.txt 2>&1
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_run.py > $OUT/${T}_sanitizer_$tool.txt 2>&1; echo "rc=$?" >> $OUT/${T}_sanitizer_$tool.txt; done
timeout 600 python bench.py --hybrid --hybrid-last 5,6 --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid56.json 2> $OUT/${T}_hybrid56.err
timeout 600 python bench.py --hybrid --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid32.json 2> $OUT/${T}_hybrid32.err
echo done
