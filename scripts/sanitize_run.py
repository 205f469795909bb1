"""Small APS syncs through every path (fused, separate calls, simulated ring), for compute-sanitizer
(memcheck, racecheck, synccheck, initcheck).  Run on the GPU box:
  compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthetic
import paper_1911_08907_b200 as aps

numels = synthetic.C1_NUMELS + [1000, 1, 130, 8195]
grads = synthetic.make_grads(numels, 2)
for engine in ("default",):
    for (e, m) in [(5, 2), (3, 0), (5, 6)]:
        g = [torch.from_numpy(a).cuda() for a in grads[0]]
        ctx = aps.ApsContext(e, m, numels)
        out = [torch.empty_like(x) for x in g]
        ctx.sync_out(g, out)                       # fused
        ctx.layer_scales(g)
        ctx.quantize_pack(g)
        ctx.allreduce()
        ctx.unscale(out)
        assert ctx.status_sync() == 0
        ctxs = [aps.ApsContext(e, m, numels, world_size=2, rank=r) for r in range(2)]
        dev = [[torch.from_numpy(a).cuda() for a in grads[r]] for r in range(2)]
        aps.sim_layer_scales(ctxs, dev)
        for r in range(2):
            ctxs[r].quantize_pack(dev[r])
        aps.sim_allreduce(ctxs)
        for r in range(2):
            ctxs[r].unscale(dev[r])
        torch.cuda.synchronize()
        print(engine, (e, m), "ok", flush=True)
