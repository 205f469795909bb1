"""Per-CTA timeline of the fused N = 1 kernel on the bench workload: start / end
stamps, quantise-item waits (count, time) and items per CTA.  Needs a build with
-DAPS_FUSED_FLAGS=80 (flag 16 = timeline):
  APS_BUILD_OUT=paper_1911_08907_b200/libaps_tl.so APS_NVCC_EXTRA=-DAPS_FUSED_FLAGS=80 \
      python -m paper_1911_08907_b200.build
  APS_LIB=paper_1911_08907_b200/libaps_tl.so python scripts/timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthetic
from paper_1911_08907_b200 import ApsContext

numels = synthetic.RESNET50_NUMELS
S = 3
sets = []
for s in range(S):
    g = [torch.from_numpy(synthetic.layer_grad(0, l, n)).cuda() for l, n in enumerate(numels)]
    sets.append((g, [torch.empty_like(x) for x in g]))
ctx = ApsContext(5, 2, numels)
for k in range(6):
    ctx.sync_out(*sets[k % S])
torch.cuda.synchronize()
for rep in range(4):
    for k in range(5):               # steady state: the previous syncs' write-backs are in flight
        ctx.sync_out(*sets[k % S])
    ctx.sync_out(*sets[rep % S])
    torch.cuda.synchronize()
    tl = ctx.timeline().astype(np.int64)
    tl = tl[tl[:, 0] > 0]
    t0 = tl[:, 0].min()
    st, en = (tl[:, 0] - t0) / 1e3, (tl[:, 3] - t0) / 1e3
    wait_us = tl[:, 1] / 1e3
    waits, items = tl[:, 2] >> 32, tl[:, 2] & 0xffffffff
    q = lambda a: f"min {a.min():6.2f} med {np.median(a):6.2f} max {a.max():6.2f}"
    print(f"rep {rep}: CTAs {len(tl)} start [{q(st)}] end [{q(en)}] us; thread-0 waits/CTA [{q(waits)}] "
          f"wait us/CTA [{q(wait_us)}] sum {wait_us.sum():.0f}; items/CTA [{q(items)}]")
