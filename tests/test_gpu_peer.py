"""Parity of the peer-memory transport (aps_peer.cu, aps_sim_connect) with the
CPU oracle, bit-exact: the flat ring order against oracle.aps_sync (the
same codes the NCCL ring produces), the hierarchical order (NEXT-3, reading
A23) and the accumulator variants (NEXT-4, reading A24) against
oracle.aps_sync_ex, per-layer formats against oracle.aps_sync_mixed, and the
Eq. (5) metric (reading A25).  p simulated ranks on one B200: every rank's
"peer" pointers are the other ranks' workspaces, the kernels and epoch flags
are the ones a multi-GPU run uses.  Needs a B200."""
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


def _to_dev(grads):
    return [[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in r] for r in grads]


def run_peer(aps, grads, e, m, hw=True, average=1, group_k=1, acc=None, kahan=False, formats=None, repeat=1,
             ctxs=None):
    p = len(grads)
    numels = [a.size for a in grads[0]]
    if ctxs is None:
        ctxs = [aps.ApsContext(e, m, numels, world_size=p, rank=r, hw_convert=hw, formats=formats)
                for r in range(p)]
        aps.sim_connect(ctxs)
        for c in ctxs:
            c.set_reduction(group_k, acc, kahan)
    for _ in range(repeat):
        dev = _to_dev(grads)
        aps.sim_layer_scales(ctxs, dev)
        for r in range(p):
            ctxs[r].quantize_pack(dev[r])
        packed = [c.packed().cpu().numpy().copy() for c in ctxs]
        aps.sim_allreduce(ctxs)
        reduced = [c.packed().cpu().numpy() for c in ctxs]
        for r in range(1, p):
            assert np.array_equal(reduced[r], reduced[0]), f"rank {r} differs after the fused all-gather"
        for r in range(p):
            ctxs[r].unscale(dev[r], average=bool(average))
        outs = [[t.cpu().numpy() for t in dev[r]] for r in range(p)]
        for r in range(1, p):
            for a, b in zip(outs[r], outs[0]):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        assert all(c.status_sync() == 0 for c in ctxs)
    return ctxs[0].scales(), packed, reduced[0], outs[0], ctxs


def compare(got, ref):
    ft, packed, reduced, outs, _ = got
    assert ref.rc == 0
    assert np.array_equal(ft, ref.ftilde), "f~ differs"
    for r in range(len(packed)):
        assert np.array_equal(packed[r], ref.packed[r]), f"rank {r} packed codes differ"
    if not np.array_equal(reduced, ref.reduced):
        bad = np.nonzero(reduced != ref.reduced)[0]
        raise AssertionError(f"reduced codes differ at bytes {bad[:8]} ({bad.size} bytes)")
    for l, (a, b) in enumerate(zip(outs, ref.out)):
        if not np.array_equal(a.view(np.uint32), b.view(np.uint32)):
            bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
            raise AssertionError(f"layer {l} outputs differ at {bad[:8]}: {a[bad[:4]]} vs {b[bad[:4]]}")


FLAT_FORMATS = [((5, 2), True), ((5, 2), False), ((4, 3), True), ((3, 0), False), ((5, 6), False),
                ((5, 10), True), ((8, 7), True), ((8, 23), True), ((6, 9), False), ((2, 1), False)]
NUMELS = synthetic.C1_NUMELS + [1000, 1, 130, 9408]


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("fmt,hw", FLAT_FORMATS, ids=lambda x: str(x))
def test_peer_flat_equals_ring_oracle(aps, orc, fmt, hw, p):
    """Flat order through peer memory == the ring oracle (O8) bit for bit."""
    e, m = fmt
    grads = synthetic.make_grads(NUMELS, p)
    compare(run_peer(aps, grads, e, m, hw), orc.aps_sync(grads, e, m, average=1))


@pytest.mark.parametrize("p", [2, 3, 5])
def test_peer_edge_cases(aps, orc, p):
    for (e, m), hw in [((5, 2), True), ((3, 0), False), ((8, 23), False)]:
        g = synthetic.edge_case_layers(p)
        compare(run_peer(aps, g, e, m, hw), orc.aps_sync(g, e, m, average=1))


def test_peer_repeated_calls(aps, orc):
    """Epoch flags and E slots advance across calls (parity-buffered slots)."""
    p = 4
    numels = NUMELS
    ctxs = None
    for it in range(4):
        grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 100 + it)
        got = run_peer(aps, grads, 5, 2, True, ctxs=ctxs)
        ctxs = got[4]
        compare(got, orc.aps_sync(grads, 5, 2, average=1))


HIER = [(4, 2), (6, 2), (6, 3), (8, 2), (8, 4), (12, 4), (16, 4), (16, 8)]


@pytest.mark.parametrize("p,k", HIER)
@pytest.mark.parametrize("fmt,hw", [((5, 2), True), ((4, 3), False), ((3, 0), False), ((5, 6), False)],
                         ids=lambda x: str(x))
def test_peer_hierarchical(aps, orc, fmt, hw, p, k):
    e, m = fmt
    grads = synthetic.make_grads(NUMELS, p, seed=synthetic.SEED + 13 * p + k)
    compare(run_peer(aps, grads, e, m, hw, group_k=k), orc.aps_sync_ex(grads, e, m, average=1, group_k=k))


ACC = [((5, 2), 8, 1, (5, 10), 0), ((5, 2), 8, 1, (8, 23), 0), ((5, 2), 8, 4, (8, 7), 0),
       ((4, 3), 4, 1, (5, 10), 0), ((5, 2), 8, 1, (5, 2), 1), ((5, 2), 8, 2, (5, 2), 1),
       ((4, 3), 6, 3, (4, 3), 1), ((5, 2), 8, 1, (5, 10), 1), ((3, 0), 4, 1, (3, 4), 1),
       ((5, 6), 4, 2, (8, 23), 1), ((5, 10), 8, 2, (8, 23), 0)]


@pytest.mark.parametrize("fmt,p,k,acc,kahan", ACC, ids=lambda x: str(x))
def test_peer_accumulators(aps, orc, fmt, p, k, acc, kahan):
    e, m = fmt
    grads = synthetic.make_grads(NUMELS, p, seed=synthetic.SEED + 5 * p + k)
    compare(run_peer(aps, grads, e, m, True, group_k=k, acc=acc, kahan=bool(kahan)),
            orc.aps_sync_ex(grads, e, m, average=1, group_k=k, acc=acc, kahan=kahan))


def test_peer_all_equal_16(aps):
    """The hand-derived sums of tests/test_oracle_order.py on the device:
    16 ranks of [1.0] in (5,2): flat 0.5, groups of 4 1.0, Kahan 1.0."""
    g = [[np.array([1.0], np.float32)] for _ in range(16)]
    for k, acc, kahan, want in [(1, None, False, 0.5), (4, None, False, 1.0), (1, None, True, 1.0),
                                (1, (5, 10), False, 1.0)]:
        out = run_peer(aps, g, 5, 2, True, group_k=k, acc=acc, kahan=kahan)[3]
        assert out[0][0] == np.float32(want), (k, acc, kahan)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_peer_mixed_formats(aps, orc, p):
    """Per-layer formats (hybrid precision) through the peer transport."""
    rng = np.random.default_rng([synthetic.SEED, 77, p])
    pool = [(5, 2), (4, 3), (3, 0), (5, 10), (8, 7), (8, 23), (5, 6)]
    fmts = [pool[i] for i in rng.integers(0, len(pool), len(NUMELS))]
    grads = synthetic.make_grads(NUMELS, p)
    compare(run_peer(aps, grads, 5, 2, True, formats=fmts), orc.aps_sync_mixed(grads, fmts, average=1))


def test_peer_resnet50_p8_full(aps, orc):
    """Config 2 at p = 8 through the peer transport, full size."""
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 8)
    compare(run_peer(aps, grads, 5, 2, True), orc.aps_sync(grads, 5, 2, average=1))


def test_peer_resnet50_p8_hierarchical_k4(aps, orc):
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 8)
    compare(run_peer(aps, grads, 5, 2, True, group_k=4), orc.aps_sync_ex(grads, 5, 2, average=1, group_k=4))


def test_reduction_argument_errors(aps):
    numels = [1000]
    ctxs = [aps.ApsContext(5, 2, numels, world_size=4, rank=r) for r in range(4)]
    with pytest.raises(aps.ApsError):
        ctxs[0].set_reduction(3)                                  # must divide p
    with pytest.raises(aps.ApsError):
        ctxs[0].set_reduction(1, acc=(4, 3))                      # narrower than the wire format
    mixed = aps.ApsContext(5, 2, [100, 100], world_size=2, rank=0, formats=[(5, 2), (8, 23)])
    with pytest.raises(aps.ApsError):
        mixed.set_reduction(1, acc=(8, 23))                       # accumulator needs one format
    # a non-flat order without the peer transport is refused at the all-reduce
    for c in ctxs:
        c.set_reduction(2)
    dev = _to_dev(synthetic.make_grads(numels, 4))
    aps.sim_layer_scales(ctxs, dev)
    for r in range(4):
        ctxs[r].quantize_pack(dev[r])
    with pytest.raises(aps.ApsError):
        aps.sim_allreduce(ctxs)


def test_round_off_error_device(aps, orc):
    """Eq. (5) on the device vs the oracle (binary64 sums in different orders:
    relative tolerance 1e-12)."""
    rng = np.random.default_rng([synthetic.SEED, 5950])
    h = (rng.standard_normal(1 << 20) * 2.0 ** rng.integers(-30, 10, 1 << 20)).astype(np.float32)
    h[::17] = 0.0
    l_ = (h * (1 + rng.standard_normal(h.size) * 0.1)).astype(np.float32)
    err, cnt = aps.round_off_error(torch.from_numpy(h).cuda(), torch.from_numpy(l_).cuda())
    ref, rcnt = orc.round_off_error(h, l_)
    assert cnt == rcnt
    assert abs(err - ref) <= 1e-12 * ref


@pytest.mark.parametrize("fmt,amax", [((5, 2), 2.0 ** 14), ((4, 3), 2.0 ** 6)], ids=["e5m2", "e4m3"])
def test_peer_fp8_all_code_pairs(aps, orc, fmt, amax):
    """Every pair of finite codes with |value| <= 2^(bias-1) through the binary16
    fold of the hardware fp8 path (p = 2, f~ = 0 so the codes are the values):
    rank 0 holds value a, rank 1 value b, for all (a, b)."""
    e, m = fmt
    codes = np.arange(256, dtype=np.uint32)
    vals = orc.decode(codes, e, m)
    vals = vals[np.isfinite(vals) & (np.abs(vals) <= amax)]
    a = np.repeat(vals, vals.size).astype(np.float32)
    b = np.tile(vals, vals.size).astype(np.float32)
    grads = [[a], [b]]
    ref = orc.aps_sync(grads, e, m, average=0)
    assert ref.ftilde[0] == 0
    compare(run_peer(aps, grads, e, m, True, average=0), ref)


@pytest.mark.parametrize("fmt", [(2, 0), (3, 2), (4, 4), (5, 6), (4, 8), (6, 9), (8, 10), (8, 20)],
                         ids=lambda f: f"b{1 + f[0] + f[1]}")
def test_peer_every_width(aps, orc, fmt):
    """Register-packed (b <= 16) and shared-memory (b > 16) widths through the
    owner-computes peer reduce, flat and hierarchical orders."""
    e, m = fmt
    grads = synthetic.make_grads(NUMELS + [8195], 4)
    compare(run_peer(aps, grads, e, m, False), orc.aps_sync(grads, e, m, average=1))
    compare(run_peer(aps, grads, e, m, False, group_k=2), orc.aps_sync_ex(grads, e, m, average=1, group_k=2))
