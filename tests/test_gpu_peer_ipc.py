"""The peer transport across PROCESSES: two ranks, each its own process and
CUDA context, exchange CUDA IPC handles of their workspaces over a gloo
group (aps_peer_export / aps_peer_import), then run aps_sync with no NCCL at
all -- the code path a multi-GPU run takes, except that both processes share
one B200 (kernels of two contexts time-slice, so the epoch-flag waits cross a
context switch).  Results bit-exact against the oracle.  Needs a B200."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import synthetic

pytestmark = pytest.mark.gpu

NUMELS = synthetic.C1_NUMELS + [1000, 1, 130]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, group_k, iters, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        import paper_1911_08907_b200 as aps
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ctx = aps.ApsContext(5, 2, NUMELS, world_size=world, rank=rank)
        ctx.connect_peers()
        ctx.set_reduction(group_k)
        outs = []
        for it in range(iters):
            grads = synthetic.make_grads(NUMELS, world, seed=synthetic.SEED + it)
            dev = [torch.from_numpy(a).cuda() for a in grads[rank]]
            ctx.sync(dev, average=True)
            st = ctx.status_sync()
            outs.append((st, ctx.scales(), ctx.packed().cpu().numpy().copy(), [t.cpu().numpy() for t in dev]))
        # the same sync captured in a CUDA graph (device-resident epochs): replays stay exact
        st = torch.cuda.Stream()
        gctx = aps.ApsContext(5, 2, NUMELS, world_size=world, rank=rank, stream=st)
        gctx.connect_peers()
        gctx.set_reduction(group_k)
        gdev = [torch.zeros(n, device="cuda") for n in NUMELS]
        graph = gctx.capture_sync(gdev)
        for it in range(iters):
            grads = synthetic.make_grads(NUMELS, world, seed=synthetic.SEED + it)
            for t, a in zip(gdev, grads[rank]):
                t.copy_(torch.from_numpy(a))
            torch.cuda.synchronize()
            dist.barrier()
            graph.replay()
            torch.cuda.synchronize()
            outs[it] = outs[it] + ([t.cpu().numpy() for t in gdev], gctx.status_sync())
        dist.barrier()           # nobody unmaps a workspace a peer may still touch
        gctx.close()
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, outs))
    except Exception as exc:      # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world,group_k", [(2, 1), (4, 2)])
def test_peer_transport_two_processes(orc, world, group_k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    iters = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, group_k, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    try:
        for _ in range(world):
            rank, res = q.get(timeout=240)
            results[rank] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert not isinstance(results[r], str), results[r]
    for it in range(iters):
        grads = synthetic.make_grads(NUMELS, world, seed=synthetic.SEED + it)
        ref = orc.aps_sync_ex(grads, 5, 2, average=1, group_k=group_k)
        for r in range(world):
            st, ft, packed, outs, gouts, gst = results[r][it]
            assert st == 0 and gst == 0
            for a, b in zip(gouts, ref.out):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
            assert np.array_equal(ft, ref.ftilde)
            assert np.array_equal(packed, ref.reduced)
            for a, b in zip(outs, ref.out):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _straggler_worker(rank, port, q, ev):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), APS_PEER_TIMEOUT_S="1")
        import torch
        import torch.distributed as dist
        import paper_1911_08907_b200 as aps
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        ctx = aps.ApsContext(5, 2, NUMELS, world_size=2, rank=rank)
        ctx.connect_peers()
        res = None
        if rank == 0:   # rank 1 never joins the sync: every wait gives up after 1 s
            dev = [torch.from_numpy(a).cuda() for a in synthetic.make_grads(NUMELS, 2)[0]]
            ctx.sync(dev)
            res = ctx.status_sync()
            ev.set()
        else:
            ev.wait(120)   # stay alive (its workspace stays mapped) until rank 0 is done
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as exc:      # pragma: no cover
        q.put((rank, repr(exc)))


def test_peer_wait_times_out_on_a_missing_rank():
    """A rank that never arrives: the waiting rank's device waits are bounded
    (APS_PEER_TIMEOUT_S) and aps_status_sync reports APS_ERR_STATE (7)."""
    ctx = mp.get_context("spawn")
    q, ev = ctx.Queue(), ctx.Event()
    port = _free_port()
    procs = [ctx.Process(target=_straggler_worker, args=(r, port, q, ev)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(2):
            r, res = q.get(timeout=240)
            got[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert got[0] == 7, got
