#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "every_width or resnet50_full or c1_and_edges" > $OUT/r02b_parity.log 2>&1; echo "rc=$?" >> $OUT/r02b_parity.log
timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_ddp.py -x -q > $OUT/r02b_peer_ddp.log 2>&1; echo "rc=$?" >> $OUT/r02b_peer_ddp.log
timeout 600 python bench.py --formats 3,0:5,2:4,3:5,6:5,10 > $OUT/r02b_bench.json 2> $OUT/r02b_bench.err
timeout 900 python scripts/ddp_step.py > $OUT/r02b_ddp_step.json 2> $OUT/r02b_ddp_step.err
bash scripts/profile.sh r02b > $OUT/r02b_profile.log 2>&1
echo done
