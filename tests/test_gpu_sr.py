"""Stochastic rounding on the device (aps_set_rounding, reading A26) against
the oracle, bit-exact: the SR Cast over fp32 probe patterns (midpoints, +-1 ulp,
subnormals, Inf/NaN, every binade), and whole syncs at p = 1 and through the
peer transport (flat and hierarchical orders).  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic
from test_gpu_peer import _to_dev, compare

pytestmark = pytest.mark.gpu

FORMATS = [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10), (8, 7), (2, 1), (6, 9), (8, 23), (4, 0)]


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


@pytest.mark.parametrize("fmt", FORMATS, ids=str)
def test_sr_cast_probes(aps, orc, fmt):
    e, m = fmt
    x = synthetic.fp32_probe_patterns(200_000)
    for seed, phase in [(0, 0), (0xDEADBEEF, 3), (2 ** 63 + 5, 1000)]:
        got = aps.debug_cast_sr(torch.from_numpy(x).cuda(), e, m, seed, phase).cpu().numpy().view(np.uint32)
        ref = orc.cast_sr(x, e, m, seed, phase)
        fin = np.isfinite(x)
        bad = np.nonzero(got[fin] != ref[fin])[0]
        assert bad.size == 0, (x[fin][bad[:5]], got[fin][bad[:5]], ref[fin][bad[:5]])
        # non-finite inputs: Inf -> Inf code, NaN -> a NaN code (same as the RNE cast)
        nf = ~fin
        assert np.array_equal(got[nf], ref[nf])


def _run(aps, grads, e, m, seed, group_k=1):
    p = len(grads)
    numels = [a.size for a in grads[0]]
    if p == 1:
        ctx = aps.ApsContext(e, m, numels)
        ctx.set_rounding(True, seed)
        dev = _to_dev(grads)
        ctx.layer_scales(dev[0])
        ctx.quantize_pack(dev[0])
        packed = [ctx.packed().cpu().numpy().copy()]
        ctx.allreduce()
        ctx.unscale(dev[0])
        assert ctx.status_sync() == 0
        out = [t.cpu().numpy() for t in dev[0]]
        return ctx.scales(), packed, ctx.packed().cpu().numpy(), out, [ctx]
    ctxs = [aps.ApsContext(e, m, numels, world_size=p, rank=r) for r in range(p)]
    aps.sim_connect(ctxs)
    for c in ctxs:
        c.set_reduction(group_k)
        c.set_rounding(True, seed)
    dev = _to_dev(grads)
    aps.sim_layer_scales(ctxs, dev)
    for r in range(p):
        ctxs[r].quantize_pack(dev[r])
    packed = [c.packed().cpu().numpy().copy() for c in ctxs]
    aps.sim_allreduce(ctxs)
    reduced = [c.packed().cpu().numpy() for c in ctxs]
    for r in range(1, p):
        assert np.array_equal(reduced[r], reduced[0])
    for r in range(p):
        ctxs[r].unscale(dev[r])
    assert all(c.status_sync() == 0 for c in ctxs)
    return ctxs[0].scales(), packed, reduced[0], [t.cpu().numpy() for t in dev[0]], ctxs


NUMELS = synthetic.C1_NUMELS + [1000, 1, 130]


@pytest.mark.parametrize("p,k", [(1, 1), (2, 1), (3, 1), (4, 1), (8, 1), (4, 2), (8, 4), (6, 3)])
@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10)], ids=str)
def test_sr_sync(aps, orc, fmt, p, k):
    e, m = fmt
    seed = 0x5EED0000 + 31 * p + k
    grads = synthetic.make_grads(NUMELS, p, seed=synthetic.SEED + 3 * p)
    # the first sync after set_rounding(seed) draws with key SplitMix64(seed, 0) (reading A27)
    compare(_run(aps, grads, e, m, seed, k),
            orc.aps_sync_ex(grads, e, m, average=1, group_k=k, sr=1, seed=orc.splitmix64(seed, 0)))


@pytest.mark.parametrize("p", [1, 3])
def test_sr_edge_cases(aps, orc, p):
    for (e, m) in [(5, 2), (3, 0), (8, 7)]:
        g = synthetic.edge_case_layers(p)
        compare(_run(aps, g, e, m, 77), orc.aps_sync_ex(g, e, m, average=1, sr=1, seed=orc.splitmix64(77, 0)))


def test_sr_argument_errors(aps):
    ctx = aps.ApsContext(5, 2, [100], world_size=2, rank=0)
    ctx.set_reduction(1, acc=(5, 10))
    with pytest.raises(aps.ApsError):
        ctx.set_rounding(True, 1)                 # not with a wider accumulator
    mixed = aps.ApsContext(5, 2, [100, 100], formats=[(5, 2), (8, 23)])
    with pytest.raises(aps.ApsError):
        mixed.set_rounding(True, 1)               # one format only


@pytest.mark.parametrize("p", [1, 4])
def test_sr_per_call_keys(aps, orc, p):
    """the k-th sync after set_rounding(seed) draws with key SplitMix64(seed, k)
    (reading A27), so repeated syncs of the SAME gradients round independently: each call
    matches the oracle run with its own key, consecutive calls differ, and re-seeding
    restarts the sequence."""
    e, m, seed = 5, 2, 1234
    grads = synthetic.make_grads(NUMELS, p, seed=synthetic.SEED + 17)
    numels = [a.size for a in grads[0]]
    if p == 1:
        ctxs = [aps.ApsContext(e, m, numels)]
    else:
        ctxs = [aps.ApsContext(e, m, numels, world_size=p, rank=r) for r in range(p)]
        aps.sim_connect(ctxs)
    for c in ctxs:
        c.set_rounding(True, seed)
    outs, prev = [], None
    for k in range(3):
        dev = _to_dev(grads)
        if p == 1:
            ctxs[0].sync(dev[0])
        else:
            aps.sim_layer_scales(ctxs, dev)
            for r in range(p):
                ctxs[r].quantize_pack(dev[r])
            aps.sim_allreduce(ctxs)
            for r in range(p):
                ctxs[r].unscale(dev[r])
        assert all(c.status_sync() == 0 for c in ctxs)
        ref = orc.aps_sync_ex(grads, e, m, average=1, sr=1, seed=orc.splitmix64(seed, k))
        got = [t.cpu().numpy() for t in dev[0]]
        for a, b in zip(got, ref.out):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        codes = ctxs[0].packed().cpu().numpy().copy()
        if prev is not None:
            assert (codes != prev).mean() > 0.1   # independent draws: many codes change
        prev = codes
        outs.append(np.concatenate(got))
    # re-seeding restarts the key sequence at k = 0
    for c in ctxs:
        c.set_rounding(True, seed)
    dev = _to_dev(grads)
    if p == 1:
        ctxs[0].sync(dev[0])
        assert np.array_equal(np.concatenate([t.cpu().numpy() for t in dev[0]]).view(np.uint32),
                              outs[0].view(np.uint32))


def test_sr_calls_round_independently(aps):
    """Per element, the rounding direction over 64 syncs of the same gradient is a
    Bernoulli draw with P(up) = (|y| - lo) / (hi - lo) (reading A26/A27): not
    the fixed per-element threshold a per-call-constant key would give."""
    n = 4096
    x = torch.full((n,), 1.3, device="cuda")       # (5,2), N = 1: y = 1.3 * 2^f~ sits at 20 % of its quantum
    ctx = aps.ApsContext(5, 2, [n])
    ctx.set_rounding(True, 99)
    ups = torch.zeros(n, device="cuda")
    for _ in range(64):
        g = x.clone()
        ctx.sync([g])
        ups += (g > 1.3).float()
    assert ctx.status_sync() == 0
    frac = (ups / 64).cpu().numpy()
    assert abs(frac.mean() - 0.2) < 0.01
    assert ((frac > 0) & (frac < 1)).mean() > 0.95
