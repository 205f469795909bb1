"""DDP communication hook with the peer transport across
two processes on one B200 (gloo process group, no NCCL): the buckets are
synchronised by libaps's owner-computes reduce over CUDA-IPC-mapped memory.
(8,23): APS is then the plain fp32 all-reduce, so every gradient must equal
fl32(g0 + g1) / 2 of the ranks' local gradients bit for bit; (5,2): both ranks
hold identical gradients within the format's resolution of the average.
Needs a B200."""
import multiprocessing as mp
import os

import numpy as np
import pytest

from test_gpu_peer_ipc import _free_port

pytestmark = pytest.mark.gpu


def _model(torch):
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 130),
                               torch.nn.ReLU(), torch.nn.Linear(130, 10)).cuda()


def _worker(rank, port, fmt, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        from paper_1911_08907_b200 import ApsHookState, aps_hook
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        e, m = fmt
        results = []
        ddp = torch.nn.parallel.DistributedDataParallel(_model(torch), bucket_cap_mb=0.05)
        state = ApsHookState(exp_bits=e, man_bits=m, transport="peer")
        ddp.register_comm_hook(state, aps_hook)
        ref = _model(torch)
        for it in range(3):   # bucket rebuild after iteration 1 re-creates the contexts
            torch.manual_seed(100 + 10 * it + rank)
            x = torch.randn(32, 64, device="cuda")
            y = torch.randint(0, 10, (32,), device="cuda")
            ddp.zero_grad()
            torch.nn.functional.cross_entropy(ddp(x), y).backward()
            torch.cuda.synchronize()
            ref.load_state_dict(ddp.module.state_dict())
            ref.zero_grad()
            torch.nn.functional.cross_entropy(ref(x), y).backward()
            local = [p.grad.detach().cpu().numpy().copy() for p in ref.parameters()]
            synced = [p.grad.detach().cpu().numpy().copy() for p in ddp.module.parameters()]
            allv = [None, None]
            dist.all_gather_object(allv, local)
            results.append((synced, allv))
            with torch.no_grad():
                for p in ddp.module.parameters():
                    p -= 0.01 * p.grad
        dist.barrier()
        state.close()
        dist.destroy_process_group()
        q.put((rank, results))
    except Exception as exc:      # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("fmt", [(8, 23), (5, 2)], ids=["fp32", "e5m2"])
def test_ddp_hook_peer_two_processes(fmt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, fmt, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(2):
            r, res = q.get(timeout=300)
            got[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(2):
        assert not isinstance(got[r], str), got[r]
    for it in range(3):
        s0, allv = got[0][it]
        s1, _ = got[1][it]
        for a, b in zip(s0, s1):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))     # identical on both ranks
        for a, g0, g1 in zip(s0, allv[0], allv[1]):
            avg = ((g0.astype(np.float32) + g1.astype(np.float32)) / np.float32(2)).astype(np.float32)
            if fmt == (8, 23):
                assert np.array_equal(a.view(np.uint32), avg.view(np.uint32))
            else:   # (5,2): 2 mantissa bits -> relative error of each code <= 2^-3 of the layer's max binade
                scale = np.abs(avg).max() + 1e-30
                assert np.abs(a - avg).max() <= 0.26 * scale
