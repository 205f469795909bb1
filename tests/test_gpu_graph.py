"""CUDA-graph capture of whole APS syncs: every kernel reads its per-call
state from device memory (64-bit wavefront claim counter -> call index and
accumulator parity, self-resetting abs-max done counter, device-resident peer
epochs), so a captured sync replays bit-exactly against the oracle with new
gradients in the same buffers.  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic
from test_gpu_peer import _to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


def _same(outs, ref):
    for a, b in zip(outs, ref.out):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("case", ["fused", "hybrid", "calls"])
def test_graph_p1(aps, orc, case):
    numels = synthetic.C1_NUMELS + [1000, 1, 130, 9408]
    fmts = [(5, 2)] * (len(numels) - 2) + [(8, 23)] * 2 if case == "hybrid" else None
    st = torch.cuda.Stream()
    ctx = aps.ApsContext(5, 2, numels, stream=st, formats=fmts)
    grads = [torch.empty(n, device="cuda") for n in numels]
    for t, a in zip(grads, synthetic.make_grads(numels, 1, seed=synthetic.SEED + 1)[0]):
        t.copy_(torch.from_numpy(a))
    torch.cuda.synchronize()
    if case == "calls":  # the separate calls (the N > 1 kernels) at p = 1
        def step():
            ctx.layer_scales(grads)
            ctx.quantize_pack(grads)
            ctx.allreduce()
            ctx.unscale(grads)
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            step()
    else:
        graph = ctx.capture_sync(grads)
    for it in range(4):
        data = synthetic.make_grads(numels, 1, seed=synthetic.SEED + 50 + it)
        for t, a in zip(grads, data[0]):
            t.copy_(torch.from_numpy(a))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        assert ctx.status_sync() == 0
        ref = orc.aps_sync_mixed(data, fmts, average=1) if fmts else orc.aps_sync(data, 5, 2, average=1)
        _same([t.cpu().numpy() for t in grads], ref)


@pytest.mark.parametrize("hybrid", [False, True], ids=["uniform", "hybrid"])
def test_graph_safe_back_to_host_mode(aps, orc, hybrid):
    """capture_sync -> replays -> set_graph_safe(False) -> plain syncs: the host-mode
    claim base must still match the 32-bit claim counter the graph-mode launches never
    touched (a drifted base decodes negative item indices)."""
    numels = synthetic.C1_NUMELS + [1000, 1, 130, 9408]
    fmts = [(5, 2)] * (len(numels) - 2) + [(8, 23)] * 2 if hybrid else None
    st = torch.cuda.Stream()
    ctx = aps.ApsContext(5, 2, numels, stream=st, formats=fmts)
    grads = [torch.empty(n, device="cuda") for n in numels]
    outs = [torch.empty(n, device="cuda") for n in numels]

    def load(seed):
        data = synthetic.make_grads(numels, 1, seed=seed)
        for t, a in zip(grads, data[0]):
            t.copy_(torch.from_numpy(a))
        torch.cuda.synchronize()
        return orc.aps_sync_mixed(data, fmts, average=1) if fmts else orc.aps_sync(data, 5, 2, average=1)

    ref = load(synthetic.SEED + 3)
    with torch.cuda.stream(st):
        ctx.sync_out(grads, outs)          # host mode first: the 32-bit counters advance
    graph = ctx.capture_sync(grads, outs)  # graph mode: priming call + capture
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    _same([t.cpu().numpy() for t in outs], ref)
    ctx.set_graph_safe(False)
    for it in range(3):
        ref = load(synthetic.SEED + 90 + it)
        with torch.cuda.stream(st):
            ctx.sync_out(grads, outs)
        torch.cuda.synchronize()
        assert ctx.status_sync() == 0
        _same([t.cpu().numpy() for t in outs], ref)
    graph2 = ctx.capture_sync(grads, outs)   # and into graph mode again
    ref = load(synthetic.SEED + 99)
    graph2.replay()
    torch.cuda.synchronize()
    assert ctx.status_sync() == 0
    _same([t.cpu().numpy() for t in outs], ref)


@pytest.mark.parametrize("p,k", [(4, 1), (8, 2)])
def test_graph_sim_peer(aps, orc, p, k):
    numels = synthetic.C1_NUMELS + [1000, 1, 130]
    st = torch.cuda.Stream()
    ctxs = [aps.ApsContext(5, 2, numels, world_size=p, rank=r, stream=st) for r in range(p)]
    aps.sim_connect(ctxs)
    for c in ctxs:
        c.set_reduction(k)
    dev = _to_dev(synthetic.make_grads(numels, p))

    def step():
        aps.sim_layer_scales(ctxs, dev)
        for r in range(p):
            ctxs[r].quantize_pack(dev[r])
        aps.sim_allreduce(ctxs)
        for r in range(p):
            ctxs[r].unscale(dev[r])

    step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        step()
    for it in range(3):
        data = synthetic.make_grads(numels, p, seed=synthetic.SEED + 70 + it)
        for r in range(p):
            for t, a in zip(dev[r], data[r]):
                t.copy_(torch.from_numpy(a))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        assert all(c.status_sync() == 0 for c in ctxs)
        ref = orc.aps_sync_ex(data, 5, 2, average=1, group_k=k)
        for r in (0, p - 1):
            _same([t.cpu().numpy() for t in dev[r]], ref)
