"""DDP communication hook on one B200: world size 1 with
the NCCL backend, a model whose parameter sizes misalign the bucket views
(so layer merging is exercised), several buckets; every parameter gradient
after backward() must equal the oracle's APS sync of the raw gradients with
the hook's layer grouping, bit for bit."""
import copy
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False], ids=["comm_stream", "same_stream"])
def test_ddp_hook_matches_oracle(pg, orc, overlap):
    import paper_1911_08907_b200 as aps
    torch.manual_seed(1)
    model = torch.nn.Sequential(torch.nn.Linear(37, 129), torch.nn.GELU(), torch.nn.Linear(129, 515),
                                torch.nn.GELU(), torch.nn.Linear(515, 3), torch.nn.LayerNorm(3)).cuda()
    ref = copy.deepcopy(model)
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[0], bucket_cap_mb=0.1)
    state = aps.ApsHookState(exp_bits=5, man_bits=2, overlap=overlap)
    ddp.register_comm_hook(state, aps.aps_hook)
    x = torch.randn(64, 37, device="cuda")
    seen_buckets = set()
    for it in range(3):
        for p in list(model.parameters()) + list(ref.parameters()):
            p.grad = None
        (ddp(x * (it + 1)).square().sum() * 1e-3).backward()
        (ref(x * (it + 1)).square().sum() * 1e-3).backward()
        torch.cuda.synchronize()
        assert state.contexts, "hook never ran"
        seen_buckets |= set(state.contexts)
        raw = {id(p): q.grad.detach().cpu().numpy().ravel() for p, q in zip(model.parameters(), ref.parameters())}
        got = {id(p): p.grad.detach().cpu().numpy().ravel() for p in model.parameters()}
        merged = 0
        for idx, groups in state.groups.items():
            params = state.bucket_params[idx]
            layers = [np.concatenate([raw[id(params[i])] for i in g]).astype(np.float32) for g in groups]
            merged += sum(len(g) > 1 for g in groups)
            res = orc.aps_sync([layers], 5, 2, average=1)
            assert res.rc == 0
            for g, out in zip(groups, res.out):
                off = 0
                for i in g:
                    n = params[i].numel()
                    assert np.array_equal(got[id(params[i])].view(np.uint32), out[off:off + n].view(np.uint32)), \
                        (idx, i)
                    off += n
        assert merged >= 1, "the misaligned parameter sizes should force at least one merged layer"
    assert len(seen_buckets) >= 2, "DDP's rebuilt buckets (bucket_cap_mb=0.1) should give several buckets"
    # overlap: the APS kernels ran on the hook's own stream, not the backward stream
    assert (state.comm_stream != torch.cuda.current_stream()) == overlap
    assert all(ent[0].stream == state.comm_stream for ent in state.contexts.values())
    state.close()
