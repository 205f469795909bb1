"""End-to-end parity of the CUDA path (libaps through the C ABI) with the CPU
oracle: scale exponents f~, every rank's packed codes, the reduced packed
codes, and the fp32 outputs -- all bit-exact (0 ulp, -0 != +0), as the
north_star requires.  Multi-rank cases use libaps's simulated-rank mode (p
virtual ranks on one B200: the same kernels and ring schedule, device copies
in place of NCCL send/recv).  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

FORMATS = [((5, 2), True), ((5, 2), False), ((4, 3), True), ((4, 3), False), ((3, 0), False),
           ((5, 6), False), ((5, 10), False), ((8, 7), False), ((8, 23), False), ((4, 6), False),
           ((6, 9), False), ((2, 1), False), ((5, 10), True), ((8, 7), True), ((8, 23), True)]
FMT_IDS = [f"e{e}m{m}{'hw' if hw else ''}" for (e, m), hw in FORMATS]


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


def _to_dev(grads):
    return [[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in r] for r in grads]


def run_gpu(aps, grads, e, m, hw, average=1, fused=False):
    """Returns (ftilde, packed per rank (after quantize), reduced, outputs) from the GPU.
    fused: p = 1 through aps_sync_out (one fused launch) instead of the four calls."""
    p = len(grads)
    numels = [a.size for a in grads[0]]
    dev = _to_dev(grads)
    if p == 1 and fused:
        ctx = aps.ApsContext(e, m, numels, hw_convert=hw)
        outs = [torch.empty_like(t) for t in dev[0]]
        ctx.sync_out(dev[0], outs, average=bool(average))
        assert ctx.status_sync() == 0
        packed = ctx.packed().cpu().numpy()
        return ctx.scales(), [packed], packed, [o.cpu().numpy() for o in outs], [ctx]
    if p == 1:
        ctx = aps.ApsContext(e, m, numels, hw_convert=hw)
        ctx.layer_scales(dev[0])
        ctx.quantize_pack(dev[0])
        packed = [ctx.packed().cpu().numpy().copy()]
        ctx.allreduce()
        outs = [torch.empty_like(t) for t in dev[0]]
        ctx.unscale(outs, average=bool(average))
        assert ctx.status_sync() == 0
        return ctx.scales(), packed, ctx.packed().cpu().numpy(), [o.cpu().numpy() for o in outs], [ctx]
    ctxs = [aps.ApsContext(e, m, numels, world_size=p, rank=r, hw_convert=hw) for r in range(p)]
    aps.sim_layer_scales(ctxs, dev)
    for r in range(p):
        ctxs[r].quantize_pack(dev[r])
    packed = [c.packed().cpu().numpy().copy() for c in ctxs]
    aps.sim_allreduce(ctxs)
    reduced = [c.packed().cpu().numpy() for c in ctxs]
    for r in range(1, p):                       # O9: every rank holds identical codes
        assert np.array_equal(reduced[r], reduced[0]), f"rank {r} differs after all-gather"
    outs = []
    for r in range(p):
        o = dev[r]                              # in place (aliases grads)
        ctxs[r].unscale(o, average=bool(average))
        outs.append([t.cpu().numpy() for t in o])
    for r in range(1, p):
        for a, b in zip(outs[r], outs[0]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert all(c.status_sync() == 0 for c in ctxs)
    return ctxs[0].scales(), packed, reduced[0], outs[0], ctxs


def check(aps, orc, grads, e, m, hw, average=1, fused=False, ref=None):
    ref = ref or orc.aps_sync(grads, e, m, average=average)
    assert ref.rc == 0
    ft, packed, reduced, outs, _ = run_gpu(aps, grads, e, m, hw, average, fused)
    assert np.array_equal(ft, ref.ftilde), "f~ differs"
    for r in range(len(grads)):
        if not np.array_equal(packed[r], ref.packed[r]):
            bad = np.nonzero(packed[r] != ref.packed[r])[0]
            raise AssertionError(f"rank {r} packed codes differ at bytes {bad[:8]}")
    if not np.array_equal(reduced, ref.reduced):
        bad = np.nonzero(reduced != ref.reduced)[0]
        raise AssertionError(f"reduced codes differ at bytes {bad[:8]} ({bad.size} bytes)")
    for l, (a, b) in enumerate(zip(outs, ref.out)):
        if not np.array_equal(a.view(np.uint32), b.view(np.uint32)):
            bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
            raise AssertionError(f"layer {l} outputs differ at {bad[:8]}: {a[bad[:4]]} vs {b[bad[:4]]}")


# ----------------------------------------------------------------- p = 1

@pytest.mark.parametrize("fused", [True, False], ids=["fused", "calls"])
@pytest.mark.parametrize("fmt,hw", FORMATS, ids=FMT_IDS)
def test_p1_c1_and_edges(aps, orc, fmt, hw, fused):
    e, m = fmt
    grads = synthetic.make_grads(synthetic.C1_NUMELS + [1000, 1, 9408, 130, 8195, 16387], 1)
    check(aps, orc, grads, e, m, hw, fused=fused)
    check(aps, orc, synthetic.edge_case_layers(1), e, m, hw, average=0, fused=fused)


@pytest.mark.parametrize("fmt,hw", [((5, 2), True), ((5, 2), False), ((3, 0), False), ((5, 6), False),
                                    ((5, 10), False), ((4, 3), True), ((5, 10), True), ((8, 23), True)], ids=lambda x: str(x))
def test_p1_resnet50_full(aps, orc, fmt, hw):
    """Config 2 at N = 1 (the bench workload, bench's launch configuration:
    the fused single launch), 161 tensors, 25,557,032 elements; also the
    four separate calls."""
    e, m = fmt
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 1)
    ref = orc.aps_sync(grads, e, m, average=1)
    check(aps, orc, grads, e, m, hw, fused=True, ref=ref)
    check(aps, orc, grads, e, m, hw, fused=False, ref=ref)


@pytest.mark.timeout(300)
def test_p1_fused_repeated_resnet50(aps, orc):
    """Many fused syncs on one context at bench scale: the monotone claim /
    completion counters must stay in step across calls (a drift hangs or
    corrupts); every 5th result is compared with the oracle."""
    numels = synthetic.RESNET50_NUMELS
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    g = [torch.from_numpy(a).cuda() for a in grads[0]]
    out = [torch.empty_like(x) for x in g]
    ctx = aps.ApsContext(5, 2, numels)
    for it in range(25):
        ctx.sync_out(g, out)
        if it % 5 == 4:
            assert ctx.status_sync() == 0
            for a, b in zip(out, ref.out):
                assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32)), it


def test_p1_fused_repeated_and_inplace(aps, orc):
    """The generation-stamped fused launch: many syncs in a row (fresh data
    each time, alternating in-place and out-of-place) stay bit-exact."""
    numels = synthetic.C1_NUMELS + [77, 9408]
    ctx = aps.ApsContext(5, 2, numels)
    for it in range(6):
        grads = synthetic.make_grads(numels, 1, seed=synthetic.SEED + 100 + it)
        ref = orc.aps_sync(grads, 5, 2)
        g = [torch.from_numpy(a).cuda() for a in grads[0]]
        if it % 2:
            ctx.sync(g)
            out = g
        else:
            out = [torch.empty_like(t) for t in g]
            ctx.sync_out(g, out)
        assert ctx.status_sync() == 0
        assert np.array_equal(ctx.scales(), ref.ftilde)
        for a, b in zip(out, ref.out):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))


# ----------------------------------------------------------------- simulated ranks

@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("fmt,hw", FORMATS, ids=FMT_IDS)
def test_sim_c1(aps, orc, fmt, hw, p):
    """Config 1 (4K/64K/256K layers) plus ragged layers, p simulated ranks."""
    e, m = fmt
    grads = synthetic.make_grads(synthetic.C1_NUMELS + [1000, 1, 130], p)
    check(aps, orc, grads, e, m, hw)


@pytest.mark.parametrize("p", [2, 3, 5])
@pytest.mark.parametrize("fmt,hw", [((5, 2), True), ((3, 0), False), ((5, 6), False), ((8, 23), False)],
                         ids=lambda x: str(x))
def test_sim_edge_cases(aps, orc, fmt, hw, p):
    e, m = fmt
    check(aps, orc, synthetic.edge_case_layers(p), e, m, hw, average=1)


def test_sim_order_sensitivity(aps, orc):
    """The p = 3 input that separates ring orders (0x71 vs 0x70)."""
    g = [[np.array([1.0], np.float32)], [np.array([0.125], np.float32)], [np.array([0.125], np.float32)]]
    for hw in (True, False):
        ft, packed, reduced, outs, _ = run_gpu(aps, g, 5, 2, hw, average=0)
        assert ft[0] == 13 and reduced[0] == 0x71 and outs[0][0] == 1.25


@pytest.mark.parametrize("fmt,hw", [((5, 2), True), ((5, 2), False), ((4, 3), True)], ids=lambda x: str(x))
def test_sim_resnet50_p8_full(aps, orc, fmt, hw):
    """Config 2 at p = 8 (simulated), full size, every code and output compared."""
    e, m = fmt
    grads = synthetic.make_grads(synthetic.RESNET50_NUMELS, 8)
    check(aps, orc, grads, e, m, hw)


def test_sim_bert_large_p8_sampled(aps, orc):
    """Config 3 (BERT-large, 391 tensors, 335M elements, (4,3), p = 8) at full
    size in the launch configuration the bench uses; outputs checked on a
    sample of elements the oracle computes one by one (O3-O10 composed per
    element in the ring order of the element's chunk), plus all f~."""
    e, m, p = 4, 3, 8
    numels = synthetic.BERT_LARGE_NUMELS
    T = sum((n + 127) // 128 for n in numels)
    Tp = p * ((T + p - 1) // p)
    chunk_tiles = Tp // p
    rng = np.random.default_rng([synthetic.SEED, 3])
    ctxs = [aps.ApsContext(e, m, numels, world_size=p, rank=r) for r in range(p)]
    dev, samples, ft_ref = [[None] * len(numels) for _ in range(p)], {}, []
    tile_off = 0
    for l, n in enumerate(numels):
        idx = np.unique(np.concatenate([rng.integers(0, n, 64), [0, n - 1]]))
        Es, vals = [], []
        for r in range(p):
            g = synthetic.layer_grad(r, l, n)
            Es.append(orc.find_max_exp(g, p))
            vals.append(g[idx].copy())
            dev[r][l] = torch.from_numpy(g).cuda()
        ft_ref.append(orc.scale_exp(e, max(Es)))
        samples[l] = (idx, np.stack(vals), tile_off)
        tile_off += (n + 127) // 128
    aps.sim_layer_scales(ctxs, dev)
    for r in range(p):
        ctxs[r].quantize_pack(dev[r])
    aps.sim_allreduce(ctxs)
    assert np.array_equal(ctxs[0].scales(), np.array(ft_ref, np.int32))
    for r in range(p):
        ctxs[r].unscale(dev[r], average=True)
    torch.cuda.synchronize()
    for l, (idx, vals, toff) in samples.items():
        ft = ft_ref[l]
        q = np.stack([orc.scale_cast_n(vals[r], ft, e, m) for r in range(p)])     # O5+O6 per rank
        c = (toff + idx // 128) // chunk_tiles                                    # O7 chunk of each element
        s = np.empty(idx.size, np.uint32)
        for k in range(idx.size):                                                 # O8 in ring order
            acc = q[(c[k] + 1) % p, k]
            for j in range(2, p + 1):
                acc = orc.ring_add(int(acc), int(q[(c[k] + j) % p, k]), e, m)
            s[k] = acc
        ref = orc.unscale_n(s, ft, p, 1, e, m)                                    # O10
        for r in (0, p - 1):
            got = dev[r][l][torch.from_numpy(idx).cuda()].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), f"layer {l} rank {r}"


# ----------------------------------------------------------------- API behaviour on the device

def test_nonfinite_flag(aps):
    g = [torch.tensor([1.0, float("nan"), 2.0], device="cuda"), torch.ones(200, device="cuda")]
    ctx = aps.ApsContext(5, 2, [3, 200])
    ctx.sync(g)
    assert ctx.status_sync() == 6
    assert ctx.status_sync() == 0                     # flag cleared
    g = [torch.ones(3, device="cuda"), torch.ones(200, device="cuda")]
    ctx.sync(g)
    assert ctx.status_sync() == 0


def test_state_and_alignment_errors(aps):
    ctx = aps.ApsContext(5, 2, [256])
    g = torch.ones(260, device="cuda")
    with pytest.raises(aps.ApsError) as ei:
        ctx.quantize_pack([g[:256]])
    assert ei.value.status == 7
    with pytest.raises(aps.ApsError) as ei:
        ctx.layer_scales([g[1:257]])                  # 4-byte offset: not 16-byte aligned
    assert ei.value.status == 3
    ctx.layer_scales([g[:256]])
    with pytest.raises(aps.ApsError):
        ctx.unscale([g[:256]])                        # before quantize_pack


def test_sync_host_e2e(aps, orc):
    """aps_sync_host: host buffers in, host buffers out, bit-exact."""
    numels = synthetic.C1_NUMELS + [77]
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    ctx = aps.ApsContext(5, 2, numels)
    hin = [torch.from_numpy(a).pin_memory() for a in grads[0]]
    hout = [torch.empty_like(t).pin_memory() for t in hin]
    dev = [torch.empty(t.shape, device="cuda") for t in hin]
    ctx.sync_host(hin, dev, hout, average=True)
    torch.cuda.synchronize()
    for a, b in zip(hout, ref.out):
        assert np.array_equal(a.numpy().view(np.uint32), b.view(np.uint32))


def test_repeated_syncs_self_reset(aps, orc):
    """The per-layer abs-max / counters reset themselves: many syncs in a row
    with different data keep matching the oracle."""
    numels = [5000, 64, 70000]
    ctx = aps.ApsContext(5, 2, numels)
    for it in range(4):
        grads = synthetic.make_grads(numels, 1, seed=synthetic.SEED + it)
        ref = orc.aps_sync(grads, 5, 2)
        g = [torch.from_numpy(a).cuda() for a in grads[0]]
        ctx.sync(g)
        assert np.array_equal(ctx.scales(), ref.ftilde)
        for a, b in zip(g, ref.out):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))


def test_nccl_world1_path(aps, orc):
    """A 1-rank NCCL communicator routes the sync through the real NCCL calls
    (unique id, ncclCommInitRank, int32 MAX all-reduce of E, in-place
    all-gather of the packed chunks) -- the plumbing of the N > 1 ring,
    checked bit-exactly on one GPU."""
    numels = synthetic.C1_NUMELS + [1000, 1]
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    comm = aps.nccl_comm_init(aps.nccl_unique_id(), 1, 0)
    try:
        ctx = aps.ApsContext(5, 2, numels, world_size=1, rank=0, nccl_comm=comm)
        g = [torch.from_numpy(a).cuda() for a in grads[0]]
        for _ in range(3):
            out = [torch.empty_like(x) for x in g]
            ctx.sync_out(g, out)
            assert ctx.status_sync() == 0
            assert np.array_equal(ctx.scales(), ref.ftilde)
            assert np.array_equal(ctx.packed().cpu().numpy(), ref.reduced)
            for a, b in zip(out, ref.out):
                assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))
        ctx.close()
    finally:
        aps.nccl_comm_destroy(comm)


@pytest.mark.timeout(300)
def test_p1_fused_repeated_formats(aps, orc):
    """The fused N = 1 kernel is bit-exact on edge cases and ResNet-50 at full size, in
    several formats, with repeated calls on one context."""
    for (e, m), hw in [((5, 2), True), ((5, 2), False), ((3, 0), False), ((5, 6), False), ((5, 10), False)]:
        check(aps, orc, synthetic.edge_case_layers(1), e, m, hw, average=0, fused=True)
        grads = synthetic.make_grads(synthetic.C1_NUMELS + [1000, 1, 130, 8195, 16387], 1)
        check(aps, orc, grads, e, m, hw, fused=True)
    numels = synthetic.RESNET50_NUMELS
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    g = [torch.from_numpy(a).cuda() for a in grads[0]]
    ctx = aps.ApsContext(5, 2, numels)
    for it in range(12):
        out = [torch.empty_like(x) for x in g]
        ctx.sync_out(g, out)
        if it % 4 == 3:
            assert ctx.status_sync() == 0
            for a, b in zip(out, ref.out):
                assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32)), (schedule, it)


def test_sync_host_flat_and_separate_buffers(aps, orc):
    """aps_sync_host coalesces copies of layers contiguous inside one allocation
    (flat buffers with per-layer views) and never across allocations (separate
    tensors that happen to be adjacent): both bit-exact."""
    numels = synthetic.C1_NUMELS + [1000, 4, 16384, 1024]
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    offs = np.concatenate([[0], np.cumsum(numels)])
    fi = torch.from_numpy(np.concatenate(grads[0])).pin_memory()
    fo = torch.empty_like(fi).pin_memory()
    fd = torch.empty(fi.numel(), device="cuda")
    hin = [fi[offs[l]:offs[l + 1]] for l in range(len(numels))]
    hout = [fo[offs[l]:offs[l + 1]] for l in range(len(numels))]
    dev = [fd[offs[l]:offs[l + 1]] for l in range(len(numels))]
    for layout in ("flat", "separate", "flat"):
        ctx = aps.ApsContext(5, 2, numels)
        if layout == "separate":
            hin = [torch.from_numpy(a).pin_memory() for a in grads[0]]
            hout = [torch.empty_like(t).pin_memory() for t in hin]
            dev = [torch.empty(t.shape, device="cuda") for t in hin]
        for _ in range(2):
            for h in hout:
                h.zero_()
            ctx.sync_host(hin, dev, hout, average=True)
            torch.cuda.synchronize()
            for a, b in zip(hout, ref.out):
                assert np.array_equal(a.numpy().view(np.uint32), b.view(np.uint32)), layout


# ----------------------------------------------------------------- every code width
# b = 1 + e + m from 3 to 32: b <= 16 (not 8/16) packs in registers with warp shuffles
# (runtime codec, or the compiled (3,0) / (5,6)), 17..31 through the per-warp shared-memory
# tile; 8/16/32 the direct paths.  Each through the fused launch, the separate calls and
# 3 simulated ranks (NCCL-ring schedule), with ragged layer tails.
WIDTHS = [(2, 0), (2, 1), (3, 1), (3, 2), (4, 2), (4, 3), (4, 4), (5, 4), (5, 5), (4, 8), (5, 7), (6, 7),
          (5, 9), (6, 9), (6, 10), (7, 10), (8, 10), (8, 13), (7, 17), (8, 20), (8, 22)]


@pytest.mark.parametrize("fmt", WIDTHS, ids=lambda f: f"b{1 + f[0] + f[1]}_e{f[0]}m{f[1]}")
def test_every_width(aps, orc, fmt):
    e, m = fmt
    numels = [4096, 1000, 1, 9408, 130, 8195, 65536 + 37]
    g1 = synthetic.make_grads(numels, 1)
    check(aps, orc, g1, e, m, False, fused=True)
    check(aps, orc, g1, e, m, False, fused=False)
    check(aps, orc, synthetic.make_grads(numels, 3), e, m, False)


@pytest.mark.parametrize("cap", [1, 2])
def test_p1_fused_occupancy_cap(aps, orc, cap):
    """aps_set_occupancy: the fused launch with 1 or 2 CTAs per SM (the DDP hook's
    overlap setting) gives the same bits; repeated calls keep the counters in step."""
    numels = synthetic.RESNET50_NUMELS[:60] + [1000, 1, 8195]
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    g = [torch.from_numpy(a).cuda() for a in grads[0]]
    ctx = aps.ApsContext(5, 2, numels)
    ctx.set_occupancy(cap)
    for _ in range(3):
        out = [torch.empty_like(x) for x in g]
        ctx.sync_out(g, out)
        assert ctx.status_sync() == 0
        assert np.array_equal(ctx.scales(), ref.ftilde)
        assert np.array_equal(ctx.packed().cpu().numpy(), ref.packed[0])
        for a, b in zip(out, ref.out):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))


@pytest.mark.timeout(300)
def test_p1_fused_concurrent_streams(aps, orc):
    """Two contexts' fused launches on two streams at once (a bench e2e / multi-bucket
    pattern): neither grid is fully resident while the other runs, so no CTA may wait on
    work held by a CTA that is not resident.  Both stay bit-exact with no wait timeout."""
    numels = synthetic.RESNET50_NUMELS
    grads = synthetic.make_grads(numels, 1)
    ref = orc.aps_sync(grads, 5, 2, average=1)
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs = [aps.ApsContext(5, 2, numels, stream=s) for s in streams]
    gs = [[torch.from_numpy(a).cuda() for a in grads[0]] for _ in range(2)]
    outs = [[torch.empty_like(x) for x in g] for g in gs]
    ptr_g = [aps.ApsContext.ptr_array(g) for g in gs]
    ptr_o = [aps.ApsContext.ptr_array(o) for o in outs]
    torch.cuda.synchronize()
    for _ in range(20):
        for i in range(2):
            ctxs[i].sync_out(ptr_g[i], ptr_o[i])
    torch.cuda.synchronize()
    for i in range(2):
        assert ctxs[i].status_sync() == 0
        for a, b in zip(outs[i], ref.out):
            assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))
        ctxs[i].close()
