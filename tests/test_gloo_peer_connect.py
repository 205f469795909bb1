"""Multi-process (gloo, CPU) check of the peer transport's host-side handshake
(ApsContext.connect_peers): every rank exports its workspace handle, the
(handle, offset) pairs are all-gathered, and every rank imports the full set in
rank order -- or, if any rank could not export, EVERY rank raises and nobody
maps anything (so all ranks fall back to the NCCL ring together, as
bench.py --transport auto does).  The CUDA calls are stubbed; the collective
logic is the binding's own."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, fail_rank, out):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1911_08907_b200.aps as A

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class Stub(A.ApsContext):
        def __init__(self):  # no device work
            self.world_size, self.rank, self.imported = world, rank, None

        def peer_export(self):
            if rank == fail_rank:
                raise A.ApsError(A.APS_ERR_CUDA, "cudaIpcGetMemHandle failed (stub)")
            return bytes([rank]) * A.PEER_HANDLE_BYTES, 256 * rank

        def peer_import(self, handles, offsets):
            self.imported = (list(handles), list(offsets))

    ctx = Stub()
    try:
        ctx.connect_peers()
        res = ("ok", [h[0] for h in ctx.imported[0]], ctx.imported[1])
    except A.ApsError as exc:
        res = ("err", str(exc), ctx.imported)
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fail_rank", [(2, -1), (3, -1), (2, 1), (3, 0)])
def test_connect_peers_agreement(world, fail_rank):
    mgr = mp.get_context("spawn").Manager()  # (a forked manager from a threaded process warns)
    out = mgr.dict()
    mp.spawn(_rank_main, args=(world, _free_port(), fail_rank, out), nprocs=world, join=True)
    for r in range(world):
        kind, a, b = out[r]
        if fail_rank < 0:
            assert kind == "ok" and a == list(range(world)) and b == [256 * q for q in range(world)]
        else:
            assert kind == "err" and f"ranks [{fail_rank}]" in a and b is None
