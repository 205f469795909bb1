"""NEXT-1 measurement: iteration time of a synthetic ResNet-50 DDP
training step (batch 32, 224x224 random images, SGD) with DDP's default
all-reduce vs the APS comm hook (1/5/2) with and without the comm-stream
overlap, plus a kernel timeline (torch.profiler / CUPTI) of the overlapped
hook: how much APS kernel time runs concurrently with backward kernels on
another stream.  One process per GPU under torchrun; prints one JSON line
(world 1 on one B200: the hook's cost without any communication saving)."""
import json
import os
import sys
import tempfile

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
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(local)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
torch.backends.cudnn.benchmark = True
APS_KERNELS = ("fused_", "absmax", "quant_pack", "unpack_unscale", "ring_reduce", "peer_", "apply_ptrs", "items_")


def build(hook, overlap=True, transport="nccl", cap=0):
    torch.manual_seed(0)
    model = torchvision.models.resnet50().cuda()
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    state = None
    if hook:
        state = aps.ApsHookState(exp_bits=5, man_bits=2, overlap=overlap, transport=transport, ctas_per_sm=cap)
        ddp.register_comm_hook(state, aps.aps_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.01, momentum=0.9)
    return ddp, opt, state


def step(ddp, opt, x, y):
    opt.zero_grad(set_to_none=True)
    loss = torch.nn.functional.cross_entropy(ddp(x), y)
    loss.backward()
    opt.step()


BATCH = int(os.environ.get("DDP_BATCH", "32"))


def run(hook, overlap=True, iters=30, warm=10, rounds=3, cap=0, batch=None):
    batch = batch or BATCH
    ddp, opt, state = build(hook, overlap, cap=cap)
    x = torch.randn(batch, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (batch,), device="cuda")
    for _ in range(warm):
        step(ddp, opt, x, y)
    best = []
    for _ in range(rounds):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(iters):
            step(ddp, opt, x, y)
        ev[1].record()
        torch.cuda.synchronize()
        best.append(ev[0].elapsed_time(ev[1]) / iters)
    if state:
        state.close()
    return sorted(best)[len(best) // 2]


def timeline(overlap=True, cap=0, batch=None):
    """Kernel intervals of 3 profiled iterations: APS kernels vs every other kernel, and
    how busy the GPU is at all (a launch-bound step leaves gaps the APS kernels fill)."""
    batch = batch or BATCH
    ddp, opt, state = build(True, overlap, cap=cap)
    x = torch.randn(batch, 3, 224, 224, device="cuda")
    y = torch.randint(0, 1000, (batch,), device="cuda")
    for _ in range(8):
        step(ddp, opt, x, y)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            step(ddp, opt, x, y)
        torch.cuda.synchronize()
    state.close()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    apsk = [e for e in ev if any(k in e["name"] for k in APS_KERNELS)]
    other = [e for e in ev if e not in apsk]
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in other)
    merged = []
    for a, b in iv:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    conc = 0.0
    n_conc = 0
    for e in apsk:
        a, b = e["ts"], e["ts"] + e["dur"]
        c = sum(max(0.0, min(b, y1) - max(a, x1)) for x1, y1 in merged)
        conc += c
        n_conc += c > 0
    streams = sorted({e["args"].get("stream") for e in apsk})
    allv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ev)
    busy, cur = 0.0, None
    for a, b in allv:
        if cur and a <= cur[1]:
            cur[1] = max(cur[1], b)
        else:
            if cur:
                busy += cur[1] - cur[0]
            cur = [a, b]
    if cur:
        busy += cur[1] - cur[0]
    span = allv[-1][1] - allv[0][0] if allv else 1.0
    return {"batch": batch, "gpu_busy_pct": round(100 * busy / span, 1), "aps_kernels": len(apsk), "aps_kernel_us": round(sum(e["dur"] for e in apsk), 1),
            "aps_us_concurrent_with_other_kernels": round(conc, 1), "aps_kernels_overlapping": n_conc,
            "aps_streams": streams,
            "other_streams": sorted({e["args"].get("stream") for e in other}),
            "first_aps": [{"name": e["name"][:40], "ts": e["ts"], "dur": e["dur"], "stream": e["args"].get("stream")}
                          for e in apsk[:6]]}


base = run(False)
with_aps = run(True, overlap=True)
no_ovl = run(True, overlap=False)
capped = run(True, overlap=True, cap=1)
tl = timeline(True)
tl0 = timeline(False)
tl1 = timeline(True, cap=1)
tl_big = timeline(True, cap=1, batch=128)
base_big = run(False, batch=128, iters=10, warm=4)
aps_big = run(True, overlap=True, cap=1, batch=128, iters=10, warm=4)
if rank == 0:
    print(json.dumps({"workload": "resnet50 DDP training step, batch 32/GPU, synthetic 224x224", "world": world,
                      "ms_per_iter_default_allreduce": round(base, 3),
                      "ms_per_iter_aps_hook_1_5_2_overlap": round(with_aps, 3),
                      "ms_per_iter_aps_hook_1_5_2_same_stream": round(no_ovl, 3),
                      "ms_per_iter_aps_hook_1_5_2_overlap_1cta_per_sm": round(capped, 3),
                      "aps_overhead_pct_overlap": round(100 * (with_aps / base - 1), 2),
                      "timeline_overlap": tl, "timeline_same_stream": tl0, "timeline_overlap_1cta_per_sm": tl1,
                      "batch128": {"ms_per_iter_default_allreduce": round(base_big, 3),
                                   "ms_per_iter_aps_hook_overlap_1cta_per_sm": round(aps_big, 3),
                                   "timeline": tl_big}}))
dist.destroy_process_group()
