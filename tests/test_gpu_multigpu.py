"""The N > 1 path on p REAL GPUs (one process per GPU, NCCL process group): the
NCCL send/recv ring (libaps's own communicator) and the peer-memory transport
(CUDA IPC over NVLink), each checked bit-exactly against the oracle over all p
ranks' gradients, plus `bench.py --gpus p` end to end (its line must report
parity.ok).  Skipped when the box has fewer than p GPUs (gpurun gives one; the
driver's multi-GPU runs exercise these).  Reference: P:252 (AllReduce SUM),
P:410 (ring on 8 GPUs), P:528 (2(p-1) steps)."""
import json
import multiprocessing as mp
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NUMELS = synthetic.C1_NUMELS + [1000, 1, 130, 600000]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _need(p):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < p:
        pytest.skip(f"needs {p} GPUs (this box has {n})")


def _worker(rank, world, port, fmt, group_k, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        import paper_1911_08907_b200 as aps
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        uid = [aps.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = aps.nccl_comm_init(uid[0], world, rank)
        e, m = fmt
        grads = synthetic.make_grads(NUMELS, world)
        res = {}
        for transport in ("nccl", "peer"):
            if transport == "nccl" and group_k != 1:
                continue   # hierarchical orders need the peer transport
            ctx = aps.ApsContext(e, m, NUMELS, world_size=world, rank=rank,
                                 nccl_comm=comm if transport == "nccl" else None, device=dev)
            if transport == "peer":
                ctx.connect_peers()
            ctx.set_reduction(group_k)
            outs = []
            for it in range(2):   # repeated syncs: the monotone epochs / counters stay in step
                g = [torch.from_numpy(a).to(dev) for a in grads[rank]]
                ctx.sync(g, average=True)
                outs.append((ctx.status_sync(), ctx.scales(), ctx.packed().cpu().numpy().copy(),
                             [t.cpu().numpy() for t in g]))
            dist.barrier()
            ctx.close()
            res[transport] = outs
        aps.nccl_comm_destroy(comm)
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("fmt,group_k", [((5, 2), 1), ((4, 3), 1), ((3, 0), 1), ((5, 2), 2)],
                         ids=["e5m2", "e4m3", "e3m0", "e5m2-k2"])
def test_multigpu_transports_bit_exact(orc, p, fmt, group_k):
    _need(p)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, p, port, fmt, group_k, q)) for r in range(p)]
    for pr in procs:
        pr.start()
    results = {}
    try:
        for _ in range(p):
            rank, res = q.get(timeout=600)
            results[rank] = res
    finally:
        for pr in procs:
            pr.join(timeout=60)
            if pr.is_alive():
                pr.kill()
    for r in range(p):
        assert not isinstance(results[r], str), results[r]
    grads = synthetic.make_grads(NUMELS, p)
    ref = orc.aps_sync_ex(grads, fmt[0], fmt[1], average=1, group_k=group_k)
    for transport in results[0]:
        for r in range(p):
            for st, ft, packed, outs in results[r][transport]:
                assert st == 0, (transport, r)
                assert np.array_equal(ft, ref.ftilde), (transport, r)
                assert np.array_equal(packed, ref.reduced), (transport, r)
                for a, b in zip(outs, ref.out):
                    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (transport, r)


@pytest.mark.parametrize("p", [2, 8])
@pytest.mark.timeout(900)
def test_bench_multigpu_self_launch(p):
    """`python bench.py --gpus p` (no torchrun: it re-launches itself) runs, and its
    line carries parity.ok for every transport it checked."""
    _need(p)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(p), "--steps", "5",
                          "--warmup", "3", "--e2e-steps", "2", "--phase-steps", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=850, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == p
    assert d["parity"]["ok"], d["parity"]
    assert {c["transport"] for c in d["parity"]["checked"]} == {"peer", "nccl"}
