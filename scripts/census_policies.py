"""Underflow / overflow census of the three scaling policies of section 3.1 /
Fig. `aps_comparing` on the synthetic ResNet-50 gradients (config
2, one rank's gradients, f~ for N ranks): APS (f~ per layer), constant loss
scaling 2^K for a sweep of K, no scaling.  Runs aps_census on the device.
Usage: python scripts/census_policies.py [e,m] [N]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_08907_b200 as aps
import synthetic

e, m = map(int, (sys.argv[1] if len(sys.argv) > 1 else "5,2").split(","))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
numels = synthetic.RESNET50_NUMELS
g = [torch.from_numpy(synthetic.layer_grad(0, l, n)).cuda() for l, n in enumerate(numels)]
ctx = aps.ApsContext(e, m, numels)
# APS scale exponents for N ranks from this rank's FindMaxExp (the MAX over ranks is the
# same binade for this synthetic family): one layer_scales pass with N = 1, then shift by log2 N
ctx.layer_scales(g)
ctx.quantize_pack(g)
ft1 = ctx.scales()
lg = N.bit_length() - 1
ft = [int(f) - lg if f != 0 else 0 for f in ft1]
nz = sum(int((t != 0).sum().item()) for t in g)
rows = []
c = ctx.census(g, ft)
rows.append({"policy": f"APS (N={N})", "underflow": int(c[:, 0].sum()), "overflow": int(c[:, 1].sum())})
for K in range(-10, 31, 2):
    c = ctx.census(g, K)
    rows.append({"policy": f"loss scaling 2^{K}", "underflow": int(c[:, 0].sum()), "overflow": int(c[:, 1].sum())})
c = ctx.census(g, 0)
rows.append({"policy": "no scaling", "underflow": int(c[:, 0].sum()), "overflow": int(c[:, 1].sum())})
print(json.dumps({"format": f"1/{e}/{m}", "N": N, "nonzero_elements": nz, "rows": rows}, indent=1))
