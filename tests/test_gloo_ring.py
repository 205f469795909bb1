"""Multi-process (gloo, CPU) check of the N > 1 host logic of the packed ring.

Each of p processes plays one rank.  The ring SCHEDULE and LAYOUT come from
libaps's host-only entry points (aps_ring_step, aps_layout) -- the same
functions aps_allreduce uses to drive ncclSend/ncclRecv -- and the bytes
travel between processes with torch.distributed (gloo) send/recv; the
arithmetic on codes (scale, Cast, the re-quantising add, unscale) is the
oracle's, on the test side.  The result must equal oracle_aps_sync bit for
bit: this validates that the schedule, chunking and all-gather reproduce the
oracle's ring order (reading A14) when real messages are exchanged.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, e, m, numels, result_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1911_08907_b200 as aps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, b = world, 1 + e + m
    grads = [synthetic.layer_grad(rank, l, n) for l, n in enumerate(numels)]

    # a1 + a2: local exponents, MAX all-reduce (Alg. 1 lines 3-4)
    E = torch.tensor([oracle.find_max_exp(g, p) for g in grads], dtype=torch.int64)
    dist.all_reduce(E, op=dist.ReduceOp.MAX)
    ft = [oracle.scale_exp(e, int(x)) for x in E]

    # a3 + a4 in libaps's layout
    T, nbytes = aps.layout(p, e, m, numels)
    codes = np.zeros(T * 128, np.uint32)
    off = 0
    for l, g in enumerate(grads):
        codes[off:off + g.size] = oracle.scale_cast_n(g, ft[l], e, m)
        off += 128 * ((g.size + 127) // 128)
    packed = oracle.pack(codes, b)
    assert packed.size == nbytes
    cb = nbytes // p
    chunk_codes = T // p * 128

    # a5: reduce-scatter over the library's schedule
    for s in range(p - 1):
        send_c, recv_c = aps.ring_step(p, rank, s)
        out = torch.from_numpy(packed[send_c * cb:(send_c + 1) * cb].copy())
        inb = torch.empty(cb, dtype=torch.uint8)
        reqs = [dist.isend(out, (rank + 1) % p), dist.irecv(inb, (rank - 1) % p)]
        for r in reqs:
            r.wait()
        recv_codes = oracle.unpack(inb.numpy(), chunk_codes, b)
        own = oracle.unpack(packed[recv_c * cb:(recv_c + 1) * cb], chunk_codes, b)
        packed[recv_c * cb:(recv_c + 1) * cb] = oracle.pack(oracle.ring_add_n(recv_codes, own, e, m), b)
    # a6: all-gather (rank r owns chunk r)
    mine = torch.from_numpy(packed[rank * cb:(rank + 1) * cb].copy())
    parts = [torch.empty(cb, dtype=torch.uint8) for _ in range(p)]
    dist.all_gather(parts, mine)
    reduced = np.concatenate([t.numpy() for t in parts])

    # a7
    allc = oracle.unpack(reduced, T * 128, b)
    outs, off = [], 0
    for l, g in enumerate(grads):
        outs.append(oracle.unscale_n(allc[off:off + g.size], ft[l], p, 1, e, m))
        off += 128 * ((g.size + 127) // 128)
    np.save(os.path.join(result_dir, f"reduced_{rank}.npy"), reduced)
    np.save(os.path.join(result_dir, f"ft_{rank}.npy"), np.array(ft, np.int32))
    np.save(os.path.join(result_dir, f"out_{rank}.npy"), np.concatenate(outs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fmt", [(2, (5, 2)), (3, (5, 2)), (2, (3, 0)), (3, (5, 6))])
def test_gloo_ring_matches_oracle(orc, tmp_path, world, fmt):
    from paper_1911_08907_b200 import build
    build.build()
    e, m = fmt
    numels = [4096, 1000, 130, 1, 9408]
    mp.spawn(_rank_main, args=(world, _free_port(), e, m, numels, str(tmp_path)), nprocs=world, join=True)
    grads = synthetic.make_grads(numels, world)
    ref = orc.aps_sync(grads, e, m, average=1)
    assert ref.rc == 0
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"ft_{r}.npy"), ref.ftilde)
        assert np.array_equal(np.load(tmp_path / f"reduced_{r}.npy"), ref.reduced), f"rank {r} reduced codes"
        out = np.load(tmp_path / f"out_{r}.npy")
        assert np.array_equal(out.view(np.uint32), np.concatenate(ref.out).view(np.uint32))
