"""Per-CTA phase timeline of the fused p = 1 kernel on the bench workload
(APS_FUSED_FLAGS bit 16).  Run on the GPU box: python scripts/timeline.py [flags]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 2
os.environ["APS_FUSED_FLAGS"] = str(flags | 16)
import numpy as np
import torch

import synthetic
from paper_1911_08907_b200 import ApsContext

numels = synthetic.RESNET50_NUMELS
g = [torch.from_numpy(synthetic.layer_grad(0, l, n)).cuda() for l, n in enumerate(numels)]
out = [torch.empty_like(x) for x in g]
ctx = ApsContext(5, 2, numels)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    ctx.sync_out(g, out)
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    ctx.timeline()[:] = 0
    ctx.sync_out(g, out)
    torch.cuda.synchronize()
    tl = ctx.timeline().astype(np.int64)
    tl = tl[tl[:, 0] > 0]
    t0 = tl[:, 0].min()
    rel = (tl - t0) / 1e3
    q = lambda a: f"min {a.min():6.2f} med {np.median(a):6.2f} max {a.max():6.2f}"
    if (tl[:, 1] > 0).all():   # barrier schedule: 4 stamps
        print(f"rep {rep}: CTAs {len(tl)}  start [{q(rel[:, 0])}]  endA [{q(rel[:, 1])}]  barrier-out [{q(rel[:, 2])}]  end [{q(rel[:, 3])}] us")
        print(f"        phaseA dur [{q(rel[:, 1] - rel[:, 0])}]  wait [{q(rel[:, 2] - rel[:, 1])}]  phaseB dur [{q(rel[:, 3] - rel[:, 2])}]")
    else:                      # wavefront schedule: start / end only
        print(f"rep {rep}: CTAs {len(tl)}  start [{q(rel[:, 0])}]  end [{q(rel[:, 3])}] us")
