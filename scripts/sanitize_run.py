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
    for (e, m) in [(5, 2), (3, 0), (5, 6), (4, 6), (6, 12)]:
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
        # the peer transport (owner-computes reduce over mapped workspaces), 3 simulated ranks
        g3 = synthetic.make_grads(numels, 3)
        pc = [aps.ApsContext(e, m, numels, world_size=3, rank=r) for r in range(3)]
        aps.sim_connect(pc)
        d3 = [[torch.from_numpy(a).cuda() for a in g3[r]] for r in range(3)]
        aps.sim_layer_scales(pc, d3)
        for r in range(3):
            pc[r].quantize_pack(d3[r])
        aps.sim_allreduce(pc)
        for r in range(3):
            pc[r].unscale(d3[r])
        torch.cuda.synchronize()
        assert all(c.status_sync() == 0 for c in ctxs + pc)
        print(engine, (e, m), "ok", flush=True)
# hybrid precision: one low format + the FP32 classifier in one fused launch
fm = [(5, 2)] * (len(numels) - 1) + [(8, 23)]
g = [torch.from_numpy(a).cuda() for a in grads[0]]
hc = aps.ApsContext(5, 2, numels, formats=fm)
hc.sync(g)
torch.cuda.synchronize()
assert hc.status_sync() == 0
print("hybrid ok", flush=True)
