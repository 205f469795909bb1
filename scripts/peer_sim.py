"""p simulated ranks through the peer transport on one device (ResNet-50
shapes): times aps_sim_allreduce per rank-reduce and serves as the ncu target
for peer_reduce_*_kernel.  Usage: python scripts/peer_sim.py [p] [iters] [group_k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_08907_b200 as aps
import synthetic

p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
e, m = 5, 2
numels = synthetic.RESNET50_NUMELS
dev = torch.device("cuda", 0)
ss = torch.cuda.Stream(dev)
sim = [aps.ApsContext(e, m, numels, world_size=p, rank=r, stream=ss, device=dev) for r in range(p)]
aps.sim_connect(sim)
for c in sim:
    c.set_reduction(k)
g = [[torch.from_numpy(synthetic.layer_grad(r, l, n)).to(dev) for l, n in enumerate(numels)] for r in range(p)]
torch.cuda.synchronize()
aps.sim_layer_scales(sim, g)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for it in range(iters):
    for r in range(p):
        sim[r].quantize_pack(g[r])
    with torch.cuda.stream(ss):
        ev[0].record(ss)
        aps.sim_allreduce(sim)
        ev[1].record(ss)
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print("sim allreduce ms:", [round(t, 4) for t in ts])
assert all(c.status_sync() == 0 for c in sim)
