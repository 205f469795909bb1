"""Per-layer formats (hybrid precision; P:545 and Table
last_layer_precision P:571-584): the CUDA path built with aps_init_mixed
against oracle_aps_sync_mixed -- f~, every rank's packed codes, the reduced
codes and the fp32 outputs, bit-exact.  Formats are drawn so that ring chunk
boundaries fall inside layers and chunks mix code widths (8, 16, 32 and
n-bit).  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

MIXED_POOL = [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10), (8, 23), (2, 1), (4, 6), (6, 9)]
NUMELS = synthetic.C1_NUMELS + [1000, 1, 9408, 130, 8195, 16387]


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


def _formats(n, seed):
    rng = np.random.default_rng(seed)
    return [MIXED_POOL[i] for i in rng.integers(0, len(MIXED_POOL), n)]


def run_gpu_mixed(aps, grads, fmts, hw, average=1, fused=False, calls=1):
    p = len(grads)
    numels = [a.size for a in grads[0]]
    dev = [[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in r] for r in grads]
    if p == 1:
        ctx = aps.ApsContext(0, 0, numels, hw_convert=hw, formats=fmts)
        outs = [torch.empty_like(t) for t in dev[0]]
        for _ in range(calls):
            if fused:
                ctx.sync_out(dev[0], outs, average=bool(average))
                packed = [ctx.packed().cpu().numpy().copy()]
            else:
                ctx.layer_scales(dev[0])
                ctx.quantize_pack(dev[0])
                packed = [ctx.packed().cpu().numpy().copy()]
                ctx.allreduce()
                ctx.unscale(outs, average=bool(average))
        assert ctx.status_sync() == 0
        return ctx.scales(), packed, ctx.packed().cpu().numpy(), [o.cpu().numpy() for o in outs]
    ctxs = [aps.ApsContext(0, 0, numels, world_size=p, rank=r, hw_convert=hw, formats=fmts) for r in range(p)]
    aps.sim_layer_scales(ctxs, dev)
    for r in range(p):
        ctxs[r].quantize_pack(dev[r])
    packed = [c.packed().cpu().numpy().copy() for c in ctxs]
    aps.sim_allreduce(ctxs)
    reduced = [c.packed().cpu().numpy() for c in ctxs]
    for r in range(1, p):
        assert np.array_equal(reduced[r], reduced[0]), f"rank {r} differs after all-gather"
    outs = []
    for r in range(p):
        ctxs[r].unscale(dev[r], average=bool(average))
        outs.append([t.cpu().numpy() for t in dev[r]])
    assert all(c.status_sync() == 0 for c in ctxs)
    return ctxs[0].scales(), packed, reduced[0], outs[0]


def check_mixed(aps, orc, grads, fmts, hw=True, average=1, fused=False, calls=1):
    ref = orc.aps_sync_mixed(grads, fmts, average=average)
    assert ref.rc == 0
    ft, packed, reduced, outs = run_gpu_mixed(aps, grads, fmts, hw, average, fused, calls)
    assert np.array_equal(ft, ref.ftilde), "f~ differs"
    for r in range(len(grads)):
        if not np.array_equal(packed[r], ref.packed[r]):
            bad = np.nonzero(packed[r] != ref.packed[r])[0]
            raise AssertionError(f"rank {r} packed codes differ at bytes {bad[:8]} ({bad.size})")
    if not np.array_equal(reduced, ref.reduced):
        bad = np.nonzero(reduced != ref.reduced)[0]
        raise AssertionError(f"reduced codes differ at bytes {bad[:8]} ({bad.size} bytes)")
    for l, (a, b) in enumerate(zip(outs, ref.out)):
        if not np.array_equal(a.view(np.uint32), b.view(np.uint32)):
            bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
            raise AssertionError(f"layer {l} {fmts[l]} outputs differ at {bad[:8]}")


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("hw", [True, False], ids=["hw", "sw"])
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "calls"])
def test_p1_mixed(aps, orc, seed, hw, fused):
    grads = synthetic.make_grads(NUMELS, 1)
    check_mixed(aps, orc, grads, _formats(len(NUMELS), seed), hw=hw, fused=fused)


@pytest.mark.parametrize("fused", [True, False], ids=["fused", "calls"])
def test_p1_mixed_edge_cases(aps, orc, fused):
    grads = synthetic.edge_case_layers(1)
    check_mixed(aps, orc, grads, _formats(len(grads[0]), 11), average=0, fused=fused)


def test_p1_mixed_repeated_fused(aps, orc):
    """Several fused calls on one context: the per-group launches keep the
    wavefront claim and layer counters in step across calls."""
    grads = synthetic.make_grads(NUMELS, 1)
    check_mixed(aps, orc, grads, _formats(len(NUMELS), 4), fused=True, calls=4)


@pytest.mark.parametrize("low", [(5, 2), (4, 3)])
@pytest.mark.parametrize("fused", [True, False], ids=["fused", "calls"])
def test_p1_resnet50_hybrid(aps, orc, low, fused):
    """The paper's hybrid precision on ResNet-50 (Table
    last_layer_precision): fc weight + bias in FP32 (8, 23), the rest low."""
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 1)
    check_mixed(aps, orc, grads, synthetic.resnet50_hybrid_formats(low), fused=fused)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("seed", [1, 2])
def test_sim_mixed(aps, orc, p, seed):
    grads = synthetic.make_grads(NUMELS, p)
    check_mixed(aps, orc, grads, _formats(len(NUMELS), seed + 10 * p))


@pytest.mark.parametrize("p", [2, 3])
def test_sim_mixed_edge_cases(aps, orc, p):
    grads = synthetic.edge_case_layers(p)
    check_mixed(aps, orc, grads, _formats(len(grads[0]), 20 + p), hw=False, average=1)


@pytest.mark.timeout(600)
def test_sim_resnet50_hybrid_p8(aps, orc):
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 8)
    check_mixed(aps, orc, grads, synthetic.resnet50_hybrid_formats((4, 3)))


def test_mixed_uniform_matches_uniform_context(aps):
    """aps_init_mixed with one format everywhere = aps_init (same bytes out)."""
    numels = NUMELS
    grads = synthetic.make_grads(numels, 1)[0]
    dev = [torch.from_numpy(a).cuda() for a in grads]
    a = aps.ApsContext(5, 2, numels)
    b = aps.ApsContext(0, 0, numels, formats=[(5, 2)] * len(numels))
    oa = [torch.empty_like(t) for t in dev]
    ob = [torch.empty_like(t) for t in dev]
    a.sync_out(dev, oa)
    b.sync_out(dev, ob)
    assert torch.equal(a.packed(), b.packed())
    for x, y in zip(oa, ob):
        assert torch.equal(x.view(torch.int32), y.view(torch.int32))


@pytest.mark.parametrize("second", [(8, 23), (5, 6), (3, 0), (4, 3), (5, 10), (6, 12), (2, 1)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("hw", [True, False], ids=["hw", "gen"])
def test_p1_two_formats_single_launch(aps, orc, second, hw):
    """Exactly two formats: ONE fused launch whose second-format items switch codec in the
    kernel (binary32 through the identity codec, any other through the runtime codec),
    with the second group first, last and interleaved in layer order; repeated calls."""
    numels = NUMELS + [65536 + 37]
    for pattern in ("last", "first", "alternate"):
        if pattern == "last":
            fmts = [(5, 2)] * (len(numels) - 2) + [second] * 2
        elif pattern == "first":
            fmts = [second] * 2 + [(5, 2)] * (len(numels) - 2)
        else:
            fmts = [(5, 2) if i % 2 else second for i in range(len(numels))]
        grads = synthetic.make_grads(numels, 1)
        check_mixed(aps, orc, grads, fmts, hw=hw, fused=True, calls=2)
