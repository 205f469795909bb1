"""Table `group_size_error` trend on synthetic gradients: Eq. (5)
average round-off error of the (5,2) APS all-reduce of ResNet-50's first
convolution weight gradient (9408 elements) versus the hierarchical group size,
p simulated ranks on one B200 through the peer transport (aps_set_reduction),
the metric on the device (aps_round_off_error).  The paper's table is 256 real
nodes and real gradients; here p = 64 (the simulated-rank limit) and each rank's
gradient is a shared signal plus rank noise (mini-batch gradients).
Usage: python scripts/group_size_error.py [p] [noise]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1911_08907_b200 as aps
import synthetic

p = int(sys.argv[1]) if len(sys.argv) > 1 else 64
noise = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
n = 9408
rng = np.random.default_rng([synthetic.SEED, 586])
mu = rng.standard_normal(n).astype(np.float32)
grads = [((mu + noise * rng.standard_normal(n).astype(np.float32)) * np.float32(2.0 ** -10)).astype(np.float32)
         for _ in range(p)]
h = torch.from_numpy(np.stack(grads).astype(np.float64).mean(0).astype(np.float32)).cuda()  # high-precision average
rows = []
for fmt in [(5, 2), (4, 3)]:
    for k in [g for g in (1, 2, 4, 8, 16, 32, 64, 128, 256) if p % g == 0 and g <= p]:
        st = torch.cuda.Stream()
        ctxs = [aps.ApsContext(fmt[0], fmt[1], [n], world_size=p, rank=r, stream=st) for r in range(p)]
        aps.sim_connect(ctxs)
        for c in ctxs:
            c.set_reduction(k)
        dev = [[torch.from_numpy(g).cuda()] for g in grads]
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            aps.sim_layer_scales(ctxs, dev)
            for r in range(p):
                ctxs[r].quantize_pack(dev[r])
            aps.sim_allreduce(ctxs)
            for r in range(p):
                ctxs[r].unscale(dev[r], average=True)
        torch.cuda.synchronize()
        assert all(c.status_sync() == 0 for c in ctxs)
        err, cnt = aps.round_off_error(h, dev[0][0])
        rows.append({"format": f"1/{fmt[0]}/{fmt[1]}", "group_size": k if k not in (1, p) else f"{k} (ring)",
                     "round_off_error": round(err, 4), "elements": cnt})
        for c in ctxs:
            c.close()
print(json.dumps({"p": p, "noise": noise, "layer": "resnet50 conv1 weight (9408)", "rows": rows}, indent=1))
