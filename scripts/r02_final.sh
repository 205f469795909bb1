#!/bin/bash
# Round-2 closing check on one box: smoke, the whole GPU suite, the default bench line, the
# format sweep, and the ncu evidence (launch list + full captures) of the hot kernels.
OUT=gpurun_out
T=${1:-r02zz}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${T}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${T}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_gpu_tests.log
timeout 600 python bench.py > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 --no-cpu-baseline > $OUT/${T}_bench_formats.json 2> $OUT/${T}_bench_formats.err
timeout 600 python bench.py --hybrid --hybrid-last 5,6 --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid56.json 2> $OUT/${T}_hybrid56.err
timeout 600 python bench.py --hybrid --steps 40 --no-cpu-baseline --no-peer-sim > $OUT/${T}_hybrid32.json 2> $OUT/${T}_hybrid32.err
APS_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/${T}_n2_plumbing.json 2> $OUT/${T}_n2_plumbing.err
bash scripts/profile.sh $T > $OUT/${T}_profile.log 2>&1

rm -f gpurun_out/*.ncu-rep; du -sh gpurun_out
echo done
