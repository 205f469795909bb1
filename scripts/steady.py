"""Steady-state timing of the APS sync: K back-to-back syncs between
ONE event pair, rotating through S gradient/output sets whose total exceeds L2, so the
deferred write-backs of step k land inside step k+1.  Prints one JSON line per mode.
Usage (GPU box): python scripts/steady.py [--sets 3] [--steps 60] [--format 5,2] [--config c2]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_08907_b200 as aps  # noqa: E402
import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sets", type=int, default=3)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--format", default="5,2")
ap.add_argument("--config", default="c2")
ap.add_argument("--modes", default="fused,separate")
a = ap.parse_args()
e, m = map(int, a.format.split(","))
numels = {"c2": synthetic.RESNET50_NUMELS, "c3": synthetic.BERT_LARGE_NUMELS}[a.config]
L = sum(numels)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
host = [synthetic.layer_grad(0, l, n) for l, n in enumerate(numels)]
sets = []
for s in range(a.sets):
    g = [torch.from_numpy(x).to(dev) for x in host]
    o = [torch.empty_like(x) for x in g]
    sets.append((g, o, aps.ApsContext.ptr_array(g), aps.ApsContext.ptr_array(o)))
# one context per buffer set (stable pointers per context, as a DDP bucket's): no per-call
# pointer-table upload
ctxs = [aps.ApsContext(e, m, numels, stream=st, device=dev) for _ in range(a.sets)]
res = {}
for mode in a.modes.split(","):
    def step(k):
        _, _, g, o = sets[k % a.sets]   # pre-marshalled pointer arrays: the host stays ahead
        ctx = ctxs[k % a.sets]
        if mode == "fused":
            ctx.sync_out(g, o, average=True)
        else:
            ctx.layer_scales(g)
            ctx.quantize_pack(g)
            ctx.allreduce()
            ctx.unscale(o, average=True)
    for k in range(2 * a.sets):
        step(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(a.steps):
        step(k)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    assert all(c.status_sync() == 0 for c in ctxs)
    res[mode] = {"us": round(ms * 1e3, 2), "GBps_fp32eq": round(4 * L / (ms * 1e-3) / 1e9, 1),
                 "dram_floor_frac": round((8 * L + L * (1 + e + m) / 8) / (ms * 1e-3) / 6444.7e9, 3)}
print(json.dumps({"steady": res, "sets": a.sets, "steps": a.steps, "format": a.format, "config": a.config}))
