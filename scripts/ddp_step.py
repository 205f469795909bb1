"""NEXT-1 measurement: iteration time of a synthetic ResNet-50 DDP training step
(batch 32, 224x224 random images, SGD) with DDP's default all-reduce vs the APS
comm hook (1/5/2).  One process per GPU under torchrun (world 1 on one B200:
the hook's cost without any communication saving).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import torchvision

import paper_1911_08907_b200 as aps

rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(local)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
torch.backends.cudnn.benchmark = True


def run(hook: bool, iters=20, warm=8):
    torch.manual_seed(0)
    model = torchvision.models.resnet50().cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    state = None
    if hook:
        state = aps.ApsHookState(exp_bits=5, man_bits=2)
        ddp.register_comm_hook(state, aps.aps_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)
    x = torch.randn(32, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (32,), device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(warm + iters):
        if i == warm:
            torch.cuda.synchronize()
            ev[0].record()
        opt.zero_grad(set_to_none=True)
        loss = torch.nn.functional.cross_entropy(ddp(x), y)
        loss.backward()
        opt.step()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / iters
    if state:
        state.close()
    return ms


base = run(False)
with_aps = run(True)
if rank == 0:
    print(json.dumps({"workload": "resnet50 DDP training step, batch 32/GPU, synthetic 224x224", "world": world,
                      "ms_per_iter_default_allreduce": round(base, 3), "ms_per_iter_aps_hook_1_5_2": round(with_aps, 3)}))
dist.destroy_process_group()
