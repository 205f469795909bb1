#!/bin/bash
OUT=gpurun_out
T=${1:-r02w}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${T}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${T}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/${T}_gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/${T}_gpu_tests.log
timeout 600 python bench.py > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
timeout 600 python bench.py --impl reference > $OUT/${T}_reference.json 2> $OUT/${T}_reference.err
echo done
