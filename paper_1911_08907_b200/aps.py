"""Thin ctypes binding of libaps (include/aps.h).

Argument marshalling only: every step of the APS path runs in libaps's
sm_100a kernels (and NCCL for the collectives).  torch supplies device
memory (the workspace and gradient buffers) and streams.  There is no CPU
fallback: if libaps.so is missing or cannot be loaded, importing the
binding raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path
from typing import Sequence

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libaps.so"

APS_OK, APS_ERR_ARG, APS_ERR_FORMAT, APS_ERR_ALIGN = 0, 1, 2, 3
APS_ERR_CUDA, APS_ERR_NCCL, APS_ERR_NONFINITE, APS_ERR_STATE = 4, 5, 6, 7
STATUS_NAMES = {0: "APS_OK", 1: "APS_ERR_ARG", 2: "APS_ERR_FORMAT", 3: "APS_ERR_ALIGN",
                4: "APS_ERR_CUDA", 5: "APS_ERR_NCCL", 6: "APS_ERR_NONFINITE", 7: "APS_ERR_STATE"}

# every symbol include/aps.h declares
EXPORTS = [
    "aps_init", "aps_workspace_bytes", "aps_set_workspace", "aps_set_hw_convert",
    "aps_layer_scales", "aps_quantize_pack", "aps_allreduce", "aps_unscale", "aps_sync", "aps_sync_out",
    "aps_sync_host", "aps_status_sync", "aps_get_scales", "aps_get_packed", "aps_layout",
    "aps_ring_step", "aps_last_error", "aps_destroy", "aps_version", "aps_nccl_unique_id",
    "aps_nccl_comm_init", "aps_nccl_comm_destroy", "aps_sim_layer_scales", "aps_sim_allreduce",
    "aps_debug_cast", "aps_debug_decode", "aps_debug_ring_reduce",
    "aps_init_mixed", "aps_layout_mixed", "aps_set_reduction", "aps_peer_export", "aps_peer_import",
    "aps_sim_connect", "aps_round_off_error", "aps_census", "aps_set_rounding", "aps_debug_cast_sr",
    "aps_set_graph_safe", "aps_set_occupancy",
]
PEER_HANDLE_BYTES = 64


class ApsError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load(path: Path | str | None = None):
    """Load libaps.so (raises if it is absent: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    import os
    p = Path(path or os.environ.get("APS_LIB") or LIB_PATH)  # APS_LIB: A/B another build
    if not p.exists():
        raise ImportError(f"libaps.so not built at {p}; run __graft_entry__.build()")
    L = ctypes.CDLL(str(p))
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    pp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "aps_init": ([ctypes.POINTER(vp), i32, i32, i32, i32, i32, vp, vp, vp], i32),
        "aps_workspace_bytes": ([vp], sz),
        "aps_set_workspace": ([vp, vp, sz], i32),
        "aps_set_hw_convert": ([vp, i32], i32),
        "aps_layer_scales": ([vp, vp], i32),
        "aps_quantize_pack": ([vp, vp], i32),
        "aps_allreduce": ([vp], i32),
        "aps_unscale": ([vp, vp, i32], i32),
        "aps_sync": ([vp, vp, i32], i32),
        "aps_sync_out": ([vp, vp, vp, i32], i32),
        "aps_sync_host": ([vp, vp, vp, vp, i32], i32),
        "aps_status_sync": ([vp], i32),
        "aps_get_scales": ([vp, vp], i32),
        "aps_get_packed": ([vp, pp, ctypes.POINTER(sz)], i32),
        "aps_layout": ([i32, i32, i32, i32, vp, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "aps_ring_step": ([i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "aps_last_error": ([vp], ctypes.c_char_p),
        "aps_destroy": ([vp], i32),
        "aps_version": ([], ctypes.c_char_p),
        "aps_nccl_unique_id": ([vp, sz], i32),
        "aps_nccl_comm_init": ([pp, vp, i32, i32], i32),
        "aps_nccl_comm_destroy": ([vp], i32),
        "aps_sim_layer_scales": ([vp, i32, vp], i32),
        "aps_sim_allreduce": ([vp, i32], i32),
        "aps_debug_cast": ([vp, vp, i64, i32, i32, i32, vp], i32),
        "aps_debug_decode": ([vp, vp, i64, i32, i32, i32, vp], i32),
        "aps_debug_ring_reduce": ([vp, vp, i64, i32, i32, i32, vp], i32),
        "aps_init_mixed": ([ctypes.POINTER(vp), vp, vp, i32, i32, i32, vp, vp, vp], i32),
        "aps_layout_mixed": ([i32, i32, vp, vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64)], i32),
        "aps_set_reduction": ([vp, i32, i32, i32, i32], i32),
        "aps_peer_export": ([vp, vp, ctypes.POINTER(ctypes.c_uint64)], i32),
        "aps_peer_import": ([vp, vp, vp], i32),
        "aps_sim_connect": ([vp, i32], i32),
        "aps_round_off_error": ([vp, vp, i64, vp, vp, vp], i32),
        "aps_census": ([vp, vp, vp, vp], i32),
        "aps_set_rounding": ([vp, i32, ctypes.c_uint64], i32),
        "aps_set_graph_safe": ([vp, i32], i32),
        "aps_set_occupancy": ([vp, i32], i32),
        "aps_debug_cast_sr": ([vp, vp, i64, i32, i32, ctypes.c_uint64, ctypes.c_uint64, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name, None)
        if f is None and path is None and not os.environ.get("APS_LIB"):
            raise ImportError(f"{p} lacks {name}: rebuild (__graft_entry__.build())")
        if f is not None:  # (an APS_LIB A/B build may predate newer entry points)
            f.argtypes, f.restype = args, res
    _lib = L
    return L


def _ptr_array(ptrs: Sequence[int]):
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


def _i64_array(vals: Sequence[int]):
    return (ctypes.c_int64 * len(vals))(*vals)


def layout(world_size: int, exp_bits: int, man_bits: int, numels: Sequence[int]) -> tuple[int, int]:
    """(T', packed_bytes) of the packed layout -- host only."""
    L = load()
    T, nb = ctypes.c_int64(), ctypes.c_int64()
    st = L.aps_layout(world_size, exp_bits, man_bits, len(numels), _i64_array(numels),
                      ctypes.byref(T), ctypes.byref(nb))
    if st:
        raise ApsError(st, "aps_layout")
    return T.value, nb.value


def _i32_array(vals: Sequence[int]):
    return (ctypes.c_int32 * len(vals))(*vals)


def layout_mixed(world_size: int, numels: Sequence[int], formats: Sequence[tuple[int, int]]) -> tuple[int, int]:
    """(T', packed_bytes) with a format (exp_bits, man_bits) per layer -- host only."""
    L = load()
    T, nb = ctypes.c_int64(), ctypes.c_int64()
    st = L.aps_layout_mixed(world_size, len(numels), _i64_array(numels), _i32_array([f[0] for f in formats]),
                            _i32_array([f[1] for f in formats]), ctypes.byref(T), ctypes.byref(nb))
    if st:
        raise ApsError(st, "aps_layout_mixed")
    return T.value, nb.value


def ring_step(world_size: int, rank: int, step: int) -> tuple[int, int]:
    L = load()
    s, r = ctypes.c_int(), ctypes.c_int()
    st = L.aps_ring_step(world_size, rank, step, ctypes.byref(s), ctypes.byref(r))
    if st:
        raise ApsError(st, "aps_ring_step")
    return s.value, r.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load().aps_nccl_unique_id(buf, 128)
    if st:
        raise ApsError(st, "aps_nccl_unique_id")
    return buf.raw


def nccl_comm_init(uid: bytes, world_size: int, rank: int) -> int:
    comm = ctypes.c_void_p()
    st = load().aps_nccl_comm_init(ctypes.byref(comm), uid, world_size, rank)
    if st:
        raise ApsError(st, "aps_nccl_comm_init")
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    load().aps_nccl_comm_destroy(comm)


class ApsContext:
    """One aps_ctx plus its torch-owned workspace.

    grads are lists of torch fp32 CUDA tensors (one per layer, contiguous,
    16-byte aligned); the order fixes the packed layout.  `formats`, if
    given, is one (exp_bits, man_bits) per layer (hybrid precision,
    aps_init_mixed) and overrides exp_bits/man_bits.
    """

    def __init__(self, exp_bits: int, man_bits: int, numels: Sequence[int], world_size: int = 1,
                 rank: int = 0, nccl_comm: int | None = None, stream=None, device=None,
                 hw_convert: bool | None = None, formats: Sequence[tuple[int, int]] | None = None):
        import torch
        self.L = load()
        self.exp_bits, self.man_bits = exp_bits, man_bits
        self.numels = [int(n) for n in numels]
        self.world_size, self.rank = world_size, rank
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        self.formats = [tuple(f) for f in formats] if formats is not None else None
        if self.formats is not None:
            if len(self.formats) != len(self.numels):
                raise ValueError("formats needs one (exp_bits, man_bits) per layer")
            st = self.L.aps_init_mixed(ctypes.byref(h), _i32_array([f[0] for f in self.formats]),
                                       _i32_array([f[1] for f in self.formats]), world_size, rank,
                                       len(self.numels), _i64_array(self.numels), nccl_comm,
                                       self.stream.cuda_stream)
        else:
            st = self.L.aps_init(ctypes.byref(h), exp_bits, man_bits, world_size, rank, len(self.numels),
                                 _i64_array(self.numels), nccl_comm, self.stream.cuda_stream)
        if st:
            raise ApsError(st, "aps_init")
        self.h = h
        nbytes = self.L.aps_workspace_bytes(h)
        # torch's caching allocator returns >= 512-byte aligned blocks.  Allocated on the
        # context's stream, where every kernel that touches it runs: when the context is
        # dropped the block is recycled only after that stream's pending work
        with torch.cuda.stream(self.stream):
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        self._ws_ptr = (base + 255) // 256 * 256
        self._check(self.L.aps_set_workspace(h, self._ws_ptr, nbytes), "aps_set_workspace")
        if hw_convert is not None:
            self._check(self.L.aps_set_hw_convert(h, int(hw_convert)), "aps_set_hw_convert")
        self._keep = []

    # -------------------------------------------------------------- plumbing
    def _check(self, st: int, what: str):
        if st:
            raise ApsError(st, f"{what}: {self.L.aps_last_error(self.h).decode(errors='replace')}")

    @staticmethod
    def _ptrs(tensors):
        if isinstance(tensors, ctypes.Array):  # already marshalled (ApsContext.ptr_array)
            return tensors
        return _ptr_array([t.data_ptr() for t in tensors])

    @staticmethod
    def ptr_array(tensors):
        """Marshal a list of layer tensors once into the host pointer array the calls take
        (pass it instead of the list to skip the per-call marshalling of many layers)."""
        return _ptr_array([t.data_ptr() for t in tensors])

    def close(self):
        if getattr(self, "h", None):
            self.L.aps_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- the path
    def layer_scales(self, grads):
        self._check(self.L.aps_layer_scales(self.h, self._ptrs(grads)), "aps_layer_scales")

    def quantize_pack(self, grads):
        self._check(self.L.aps_quantize_pack(self.h, self._ptrs(grads)), "aps_quantize_pack")

    def allreduce(self):
        self._check(self.L.aps_allreduce(self.h), "aps_allreduce")

    def unscale(self, out, average: bool = True):
        self._check(self.L.aps_unscale(self.h, self._ptrs(out), int(average)), "aps_unscale")

    def sync(self, grads, average: bool = True):
        self._check(self.L.aps_sync(self.h, self._ptrs(grads), int(average)), "aps_sync")

    def sync_out(self, grads, out, average: bool = True):
        self._check(self.L.aps_sync_out(self.h, self._ptrs(grads), self._ptrs(out), int(average)), "aps_sync_out")

    def sync_host(self, host_in, dev_grads, host_out, average: bool = True):
        self._check(self.L.aps_sync_host(self.h, self._ptrs(host_in), self._ptrs(dev_grads),
                                         self._ptrs(host_out), int(average)), "aps_sync_host")

    def status_sync(self) -> int:
        return self.L.aps_status_sync(self.h)

    def scales(self):
        import numpy as np
        out = np.zeros(len(self.numels), dtype=np.int32)
        self._check(self.L.aps_get_scales(self.h, out.ctypes.data), "aps_get_scales")
        return out

    def packed(self):
        """The packed buffer as a torch uint8 view (device)."""
        import torch
        ptr, nb = ctypes.c_void_p(), ctypes.c_size_t()
        self._check(self.L.aps_get_packed(self.h, ctypes.byref(ptr), ctypes.byref(nb)), "aps_get_packed")
        off = ptr.value - self.workspace.data_ptr()
        return self.workspace[off:off + nb.value]

    def set_hw_convert(self, enable: bool):
        self._check(self.L.aps_set_hw_convert(self.h, int(enable)), "aps_set_hw_convert")

    def set_reduction(self, group_k: int = 1, acc: tuple[int, int] | None = None, kahan: bool = False):
        """Reduction order (hierarchical group size, 1 = flat ring) and accumulator
        (format, Kahan) of the all-reduce (aps_set_reduction)."""
        wire = self.formats[0] if self.formats is not None else (self.exp_bits, self.man_bits)
        ae, am = acc if acc is not None else wire
        self._check(self.L.aps_set_reduction(self.h, group_k, ae, am, int(kahan)), "aps_set_reduction")

    def capture_sync(self, grads, out=None, average: bool = True):
        """Capture one aps_sync_out (grads -> out, default in place) into a CUDA graph
        and return it; ``graph.replay()`` then re-runs the whole synchronisation on
        whatever the same buffers hold.  Every kernel takes its per-call state
        (self-resetting counters, peer epochs) from device memory, so replays are
        exact.  The context's stream must not be the legacy default stream.  One
        un-captured call first uploads the pointer tables."""
        import torch
        out = grads if out is None else out
        self.set_graph_safe(True)
        self.sync_out(grads, out, average)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self.sync_out(grads, out, average)
        return g

    def set_graph_safe(self, enable: bool = True):
        """aps_set_graph_safe: every launch is capture-safe already (recorded only)."""
        self._check(self.L.aps_set_graph_safe(self.h, int(enable)), "aps_set_graph_safe")

    def set_occupancy(self, ctas_per_sm: int = 0):
        """Cap the fused one-rank launch at ctas_per_sm CTAs per SM (0 = as many as fit),
        leaving SM resources to concurrent work on other streams (aps_set_occupancy)."""
        self._check(self.L.aps_set_occupancy(self.h, int(ctas_per_sm)), "aps_set_occupancy")

    def set_rounding(self, stochastic: bool = False, seed: int = 0):
        """Nearest-even (default) or stochastic rounding of every Cast (aps_set_rounding)."""
        self._check(self.L.aps_set_rounding(self.h, int(stochastic), seed), "aps_set_rounding")

    def census(self, grads, scale_exp):
        """Underflow / overflow counts [n_layers, 2] of Cast(g * 2^s_l) (aps_census);
        scale_exp: one exponent per layer, or one int for every layer."""
        import numpy as np
        if isinstance(scale_exp, int):
            scale_exp = [scale_exp] * len(self.numels)
        se = np.ascontiguousarray(scale_exp, dtype=np.int32)
        out = np.zeros((len(self.numels), 2), dtype=np.uint64)
        self._check(self.L.aps_census(self.h, self._ptrs(grads), se.ctypes.data, out.ctypes.data), "aps_census")
        return out

    # -------------------------------------------------------------- peer transport
    def peer_export(self) -> tuple[bytes, int]:
        buf = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
        off = ctypes.c_uint64()
        self._check(self.L.aps_peer_export(self.h, buf, ctypes.byref(off)), "aps_peer_export")
        return buf.raw, off.value

    def peer_import(self, handles: Sequence[bytes], offsets: Sequence[int]):
        blob = b"".join(handles)
        offs = (ctypes.c_uint64 * len(offsets))(*offsets)
        self._check(self.L.aps_peer_import(self.h, blob, offs), "aps_peer_import")

    def connect_peers(self, group=None):
        """Map every rank's workspace (CUDA IPC) and switch the all-reduce to the
        peer-memory transport.  Collective over the torch.distributed group."""
        import torch.distributed as dist
        try:
            mine = self.peer_export()
        except ApsError as exc:
            mine = str(exc)
        allv = [None] * self.world_size
        dist.all_gather_object(allv, mine, group=group)
        bad = [r for r, v in enumerate(allv) if not isinstance(v, tuple)]
        if bad:  # every rank takes the same decision: nobody maps anything
            raise ApsError(APS_ERR_STATE, f"aps_peer_export failed on ranks {bad}: {allv[bad[0]]}")
        self.peer_import([h for h, _ in allv], [o for _, o in allv])
        dist.barrier(group=group)


def sim_layer_scales(ctxs: Sequence[ApsContext], grads_per_rank):
    L = load()
    flat = [t for g in grads_per_rank for t in g]
    hs = _ptr_array([c.h.value for c in ctxs])
    st = L.aps_sim_layer_scales(hs, len(ctxs), _ptr_array([t.data_ptr() for t in flat]))
    if st:
        raise ApsError(st, "aps_sim_layer_scales: " + L.aps_last_error(ctxs[0].h).decode())


def sim_connect(ctxs: Sequence[ApsContext]):
    """Connect simulated ranks through the peer-memory transport (aps_sim_connect)."""
    L = load()
    hs = _ptr_array([c.h.value for c in ctxs])
    st = L.aps_sim_connect(hs, len(ctxs))
    if st:
        raise ApsError(st, "aps_sim_connect: " + L.aps_last_error(ctxs[0].h).decode())


def round_off_error(grad_h, grad_l) -> tuple[float, int]:
    """Eq. (5) on the device: mean of |(h - l) / h| over h != 0
    (binary64 sum on the GPU).  Returns (error, count)."""
    import torch
    acc = torch.zeros(2, dtype=torch.float64, device=grad_h.device)
    st = load().aps_round_off_error(grad_h.data_ptr(), grad_l.data_ptr(), grad_h.numel(), acc.data_ptr(),
                                    acc.data_ptr() + 8, torch.cuda.current_stream(grad_h.device).cuda_stream)
    if st:
        raise ApsError(st, "aps_round_off_error")
    s = float(acc[0].item())
    n = int(acc[1:].view(torch.int64).item())
    return (s / n if n else 0.0), n


def sim_allreduce(ctxs: Sequence[ApsContext]):
    L = load()
    hs = _ptr_array([c.h.value for c in ctxs])
    st = L.aps_sim_allreduce(hs, len(ctxs))
    if st:
        raise ApsError(st, "aps_sim_allreduce: " + L.aps_last_error(ctxs[0].h).decode())


def debug_cast(x, exp_bits: int, man_bits: int, hw: bool = False):
    """Device cast of an arbitrary fp32 CUDA tensor -> int32 codes tensor (test only)."""
    import torch
    out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    st = load().aps_debug_cast(x.data_ptr(), out.data_ptr(), x.numel(), exp_bits, man_bits, int(hw),
                               torch.cuda.current_stream(x.device).cuda_stream)
    if st:
        raise ApsError(st, "aps_debug_cast")
    return out


def debug_cast_sr(x, exp_bits: int, man_bits: int, seed: int, phase: int = 0):
    """Device stochastic-rounding cast of an fp32 CUDA tensor -> int32 codes (test only)."""
    import torch
    out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    st = load().aps_debug_cast_sr(x.data_ptr(), out.data_ptr(), x.numel(), exp_bits, man_bits, seed, phase,
                                  torch.cuda.current_stream(x.device).cuda_stream)
    if st:
        raise ApsError(st, "aps_debug_cast_sr")
    return out


def debug_decode(codes, exp_bits: int, man_bits: int, hw: bool = False):
    import torch
    out = torch.empty(codes.shape, dtype=torch.float32, device=codes.device)
    st = load().aps_debug_decode(codes.data_ptr(), out.data_ptr(), codes.numel(), exp_bits, man_bits,
                                 int(hw), torch.cuda.current_stream(codes.device).cuda_stream)
    if st:
        raise ApsError(st, "aps_debug_decode")
    return out


def debug_ring_reduce(own, recv, n_tiles: int, exp_bits: int, man_bits: int, hw: bool = False):
    import torch
    st = load().aps_debug_ring_reduce(own.data_ptr(), recv.data_ptr(), n_tiles, exp_bits, man_bits, int(hw),
                                      torch.cuda.current_stream(own.device).cuda_stream)
    if st:
        raise ApsError(st, "aps_debug_ring_reduce")
