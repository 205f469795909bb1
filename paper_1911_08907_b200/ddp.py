"""DDP communication hook running APS on every gradient bucket (SURVEY 8(f)
NEXT-1): DistributedDataParallel hands each bucket to `aps_hook` as soon as
backward() has produced it, so the low-precision synchronisation of early
buckets overlaps the backward pass of later layers.

Per bucket: the flat fp32 buffer is split at the parameter boundaries into
APS layers (Alg. 1's per-layer exponents); a parameter whose view
does not start 16-byte aligned is merged into the preceding layer (so the
bucket may have fewer exponents than parameters -- P:230 allows several
consecutive layers "as a whole tensor").  The buffer is synchronised in place
by libaps (scale, Cast, packed ring over NCCL -- or, with
transport="peer", the owner-computes reduce over CUDA-IPC-mapped peer memory --
unscale, average).

Overlap (APS is applied to merged buckets while the backward pass
continues): every bucket's sync runs on a dedicated communication stream that
first waits on an event of the backward (current) stream, so backward kernels
of later layers run concurrently with the APS kernels of earlier buckets, and
the peer transport's cross-rank waits never sit on the backward stream.  The
hook returns a CUDA-aware Future (devices=[dev]) completed on the comm stream:
DDP's wait() makes its own stream wait on that event, never the host.

Usage:
    state = ApsHookState(process_group=None, exp_bits=5, man_bits=2)
    ddp_model.register_comm_hook(state, aps_hook)
"""
import torch
import torch.distributed as dist

from .aps import ApsContext, nccl_comm_destroy, nccl_comm_init, nccl_unique_id


class ApsHookState:
    """Per-process hook state: the format, the NCCL communicator libaps uses
    for its ring (created here, collectively, outside backward), and one
    ApsContext per bucket (created on the bucket's first call)."""

    def __init__(self, process_group=None, exp_bits: int = 5, man_bits: int = 2, average: bool = True,
                 transport: str = "nccl", group_k: int = 1, overlap: bool = True, ctas_per_sm: int = 0):
        if transport not in ("nccl", "peer"):
            raise ValueError("transport must be 'nccl' or 'peer'")
        self.pg = process_group if process_group is not None else dist.group.WORLD
        self.exp_bits, self.man_bits, self.average = exp_bits, man_bits, average
        self.transport, self.group_k = transport, group_k
        self.overlap = overlap  # False: run on the backward stream (no overlap; A/B only)
        self.ctas_per_sm = ctas_per_sm  # occupancy cap of the one-rank fused launch (aps_set_occupancy)
        self.world = dist.get_world_size(self.pg)
        self.rank = dist.get_rank(self.pg)
        self.comm = None
        if self.world > 1 and transport == "nccl":
            uid = [nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=dist.get_global_rank(self.pg, 0), group=self.pg)
            self.comm = nccl_comm_init(uid[0], self.world, self.rank)
        self.comm_stream = None  # created on the first bucket (the bucket's device)
        self.contexts: dict = {}  # bucket index -> (ApsContext, layer spans, buffer ptr, marshalled views)
        self.groups: dict = {}  # bucket index -> parameter indices per APS layer
        self.bucket_params: dict = {}  # bucket index -> its parameters

    def close(self):
        if self.comm_stream is not None:
            self.comm_stream.synchronize()
        for ent in self.contexts.values():
            ent[0].close()
        self.contexts.clear()
        if self.comm:
            nccl_comm_destroy(self.comm)
            self.comm = None


def layer_spans(buffer: torch.Tensor, numels):
    """Split a flat bucket into APS layers at 16-byte-aligned parameter starts.
    Returns [(offset, numel)] per layer and the parameter indices of each."""
    base = buffer.data_ptr()
    spans, groups, off = [], [], 0
    for i, n in enumerate(numels):
        if not spans or (base + 4 * off) % 16 == 0:
            spans.append([off, n])
            groups.append([i])
        else:
            spans[-1][1] += n
            groups[-1].append(i)
        off += n
    return [tuple(s) for s in spans], groups


def aps_hook(state: ApsHookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    if buf.dtype != torch.float32:
        raise TypeError("aps_hook needs fp32 gradients")
    dev = buf.device
    if state.comm_stream is None:
        # high priority: the block scheduler hands freed SM slots to the APS kernels before the
        # backward kernels' remaining CTAs, so a sync runs alongside backward, not after it
        state.comm_stream = (torch.cuda.Stream(dev, priority=-1) if state.overlap
                             else torch.cuda.current_stream(dev))
    cs = state.comm_stream
    idx = bucket.index()
    entry = state.contexts.get(idx)
    if entry is None or entry[2] != buf.data_ptr() or entry[4] != buf.numel():
        numels = [p.numel() for p in bucket.parameters()]
        spans, groups = layer_spans(buf, numels)
        if entry is None or entry[1] != spans:
            if entry is not None:
                entry[0].close()
            ctx = ApsContext(state.exp_bits, state.man_bits, [n for _, n in spans], world_size=state.world,
                             rank=state.rank, nccl_comm=state.comm, stream=cs, device=dev)
            if state.world > 1 and state.transport == "peer":
                # every rank reaches this bucket's first sync together: map the workspaces
                ctx.connect_peers(group=state.pg)
            if state.group_k != 1:
                ctx.set_reduction(state.group_k)
            if state.ctas_per_sm:
                ctx.set_occupancy(state.ctas_per_sm)
        else:
            ctx = entry[0]
        views = ApsContext.ptr_array([buf[o:o + n] for o, n in spans])
        state.contexts[idx] = (ctx, spans, buf.data_ptr(), views, buf.numel())
        state.groups[idx] = groups
        state.bucket_params[idx] = list(bucket.parameters())
    ctx, views = state.contexts[idx][0], state.contexts[idx][3]
    # the bucket's gradients are complete on the backward stream: the comm stream waits
    # for them (device-side), then the APS sync runs there while backward continues
    cs.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cs):
        ctx.sync(views, average=state.average)
        buf.record_stream(cs)
        fut = torch.futures.Future(devices=[dev])
        fut.set_result(buf)   # records an event on cs; DDP's wait() waits on it device-side
    return fut
