#!/bin/bash
# A/B of the hybrid-precision (per-layer format) path: last-layer format and
# concurrent vs serial format-group launches.  Writes gpurun_out/hybrid_ab.txt.
out=gpurun_out/hybrid_ab.txt; : > $out
run() { echo "== $*" >> $out; timeout 300 env "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], {k:v['us'] for k,v in d['phases'].items()})" >> $out; }
run APS_X=1 python bench.py --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --hybrid --no-cpu-baseline --steps 300
run APS_HYBRID_FUSE=0 python bench.py --hybrid --no-cpu-baseline --steps 300
run APS_HYBRID_FUSE=0 APS_GROUP_STREAMS=0 python bench.py --hybrid --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --hybrid --format 4,3 --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --hybrid --hybrid-last 4,3 --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --hybrid --hybrid-last 5,6 --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --hybrid --hybrid-last 5,10 --no-cpu-baseline --steps 300
run APS_X=1 python bench.py --format 8,23 --no-cpu-baseline --steps 300
cat $out
