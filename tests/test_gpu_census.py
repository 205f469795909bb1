"""The underflow / overflow census on the device (aps_census) against the
oracle, for the three scaling policies of section 3.1 / Fig. `aps_comparing`:
APS (f~ per layer), constant loss scaling, no scaling.  Counts are integers:
bit-exact.  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 10)])
@pytest.mark.parametrize("numels", [synthetic.C1_NUMELS + [1000, 1, 130, 9408], synthetic.RESNET50_NUMELS],
                         ids=["c1", "resnet50"])
def test_census_policies(aps, orc, fmt, numels):
    e, m = fmt
    g = synthetic.make_grads(numels, 1)[0]
    g[0][:7] = [2.0 ** 20, -(2.0 ** 19), np.inf, np.nan, 2.0 ** -150, 3e-45, -0.0]   # overflow / non-finite / tiny
    dev = [torch.from_numpy(a).cuda() for a in g]
    ctx = aps.ApsContext(e, m, numels)
    fts = [orc.scale_exp(e, orc.find_max_exp(a[np.isfinite(a)], 1)) for a in g]
    for policy, s in [("aps", fts), ("loss-scale 2^-5", [-5] * len(g)), ("loss-scale 2^10", [10] * len(g)),
                      ("none", [0] * len(g))]:
        got = ctx.census(dev, s)
        ref = np.array([orc.census(a, int(sl), e, m) for a, sl in zip(g, s)], dtype=np.uint64)
        assert np.array_equal(got, ref), policy
    ctx.close()
