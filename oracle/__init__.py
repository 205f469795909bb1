"""CPU oracle for the APS gradient synchronisation (arXiv 1911.08907).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1911_08907_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``aps_oracle.c`` (plain C, binary64 unless the paper
fixes binary32); this module only builds it with gcc and marshals numpy
arrays through ctypes.  Every function cites the paper passage it follows in
the C source.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "aps_oracle.c"
LIB = HERE / "liboracle.so"

EMPTY = -(2**31)       # FindMaxExp of an all-zero tensor ("-INF", Alg. 1)
NONFINITE = 2**31 - 1
OK, ERR_ARG, ERR_FORMAT, ERR_NONFINITE = 0, 1, 2, 6
TILE = 128


def build(force: bool = False) -> Path:
    """Compile aps_oracle.c with gcc (IEEE binary32/64, no contraction)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-fexcess-precision=standard", "-Wall", "-Wextra",
             "-pthread", "-o", str(tmp), str(SRC), "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        i32, i64, u32, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_float
        vp = ctypes.c_void_p
        L.oracle_format_valid.argtypes = [ctypes.c_int, ctypes.c_int]
        L.oracle_bias.argtypes = [ctypes.c_int]
        L.oracle_cast1.argtypes = [f32, ctypes.c_int, ctypes.c_int]
        L.oracle_cast1.restype = u32
        L.oracle_decode1.argtypes = [u32, ctypes.c_int, ctypes.c_int]
        L.oracle_decode1.restype = f32
        L.oracle_cast.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int]
        L.oracle_decode.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int]
        L.oracle_find_max_exp.argtypes = [vp, i64, ctypes.c_int]
        L.oracle_find_max_exp.restype = i32
        L.oracle_scale_exp.argtypes = [ctypes.c_int, i32]
        L.oracle_scale_exp.restype = i32
        L.oracle_scale.argtypes = [f32, i32]
        L.oracle_scale.restype = f32
        L.oracle_ring_add.argtypes = [u32, u32, ctypes.c_int, ctypes.c_int]
        L.oracle_ring_add.restype = u32
        L.oracle_unscale1.argtypes = [u32, i32, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_unscale1.restype = f32
        L.oracle_total_tiles.argtypes = [ctypes.c_int, ctypes.c_int, vp]
        L.oracle_total_tiles.restype = i64
        L.oracle_packed_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
        L.oracle_packed_bytes.restype = i64
        L.oracle_pack.argtypes = [vp, i64, ctypes.c_int, vp]
        L.oracle_unpack.argtypes = [vp, i64, ctypes.c_int, vp]
        L.oracle_aps_sync.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                      vp, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int]
        L.oracle_ring_add_n.argtypes = [vp, vp, vp, i64, ctypes.c_int, ctypes.c_int]
        L.oracle_unscale_n.argtypes = [vp, vp, i64, i32, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_scale_cast_n.argtypes = [vp, vp, i64, i32, ctypes.c_int, ctypes.c_int]
        L.oracle_packed_bytes_mixed.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.oracle_packed_bytes_mixed.restype = i64
        L.oracle_aps_sync_mixed.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp, vp, vp]
        ci = ctypes.c_int
        u64 = ctypes.c_uint64
        L.oracle_aps_sync_ex.argtypes = [ci, ci, ci, ci, vp, vp, ci, ci, ci, ci, ci, ci, u64, vp, vp, vp, vp]
        L.oracle_splitmix64.argtypes = [u64, u64]
        L.oracle_splitmix64.restype = u64
        L.oracle_cast_sr1.argtypes = [f32, ci, ci, u32]
        L.oracle_cast_sr1.restype = u32
        L.oracle_cast_sr.argtypes = [vp, vp, i64, ci, ci, u64, u64]
        L.oracle_reduce1.argtypes = [vp, ci, i64, i64, ci, ci, ci, ci, ci, ci]
        L.oracle_reduce1.restype = u32
        L.oracle_round_off_error.argtypes = [vp, vp, i64, vp]
        L.oracle_round_off_error.restype = ctypes.c_double
        L.oracle_census.argtypes = [vp, i64, i32, ci, ci, vp, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def bias(e: int) -> int:
    return lib().oracle_bias(e)


def format_valid(e: int, m: int) -> bool:
    return lib().oracle_format_valid(e, m) == OK


def cast(x, e: int, m: int) -> np.ndarray:
    """O6: fp32 -> (e,m) codes (uint32), RNE, gradual underflow, IEEE overflow."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint32)
    rc = lib().oracle_cast(_ptr(x), _ptr(out), x.size, e, m)
    if rc:
        raise ValueError(f"oracle_cast rc={rc}")
    return out


def decode(codes, e: int, m: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    out = np.empty(c.shape, dtype=np.float32)
    rc = lib().oracle_decode(_ptr(c), _ptr(out), c.size, e, m)
    if rc:
        raise ValueError(f"oracle_decode rc={rc}")
    return out


def find_max_exp(g, N: int) -> int:
    g = np.ascontiguousarray(g, dtype=np.float32)
    return lib().oracle_find_max_exp(_ptr(g), g.size, N)


def scale_exp(e: int, E: int) -> int:
    return lib().oracle_scale_exp(e, E)


def scale(g: float, ft: int) -> float:
    return lib().oracle_scale(g, ft)


def ring_add(a: int, b: int, e: int, m: int) -> int:
    return lib().oracle_ring_add(a, b, e, m)


def ring_add_n(acc, addend, e: int, m: int) -> np.ndarray:
    a = np.ascontiguousarray(acc, dtype=np.uint32)
    b = np.ascontiguousarray(addend, dtype=np.uint32)
    out = np.empty(a.shape, dtype=np.uint32)
    lib().oracle_ring_add_n(_ptr(a), _ptr(b), _ptr(out), a.size, e, m)
    return out


def unscale_n(s, ft: int, N: int, average: int, e: int, m: int) -> np.ndarray:
    c = np.ascontiguousarray(s, dtype=np.uint32)
    out = np.empty(c.shape, dtype=np.float32)
    lib().oracle_unscale_n(_ptr(c), _ptr(out), c.size, ft, N, average, e, m)
    return out


def scale_cast_n(g, ft: int, e: int, m: int) -> np.ndarray:
    x = np.ascontiguousarray(g, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint32)
    lib().oracle_scale_cast_n(_ptr(x), _ptr(out), x.size, ft, e, m)
    return out


def unscale1(s: int, ft: int, N: int, average: int, e: int, m: int) -> float:
    return lib().oracle_unscale1(s, ft, N, average, e, m)


def total_tiles(p: int, numels) -> int:
    n = np.ascontiguousarray(numels, dtype=np.int64)
    return lib().oracle_total_tiles(p, n.size, _ptr(n))


def packed_bytes(p: int, e: int, m: int, numels) -> int:
    n = np.ascontiguousarray(numels, dtype=np.int64)
    return lib().oracle_packed_bytes(p, e, m, n.size, _ptr(n))


def pack(codes, b: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    out = np.zeros((c.size * b + 7) // 8, dtype=np.uint8)
    lib().oracle_pack(_ptr(c), c.size, b, _ptr(out))
    return out


def unpack(buf, n: int, b: int) -> np.ndarray:
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    out = np.empty(n, dtype=np.uint32)
    lib().oracle_unpack(_ptr(buf), n, b, _ptr(out))
    return out


class SyncResult:
    def __init__(self, rc, ftilde, packed, reduced, out):
        self.rc, self.ftilde, self.packed, self.reduced, self.out = rc, ftilde, packed, reduced, out


def aps_sync(grads, e: int, m: int, average: int = 1, want_packed: bool = True,
             want_out: bool = True, n_threads: int = 1) -> SyncResult:
    """Full APS sync (Alg. 1) over p simulated ranks.

    ``grads[r][l]`` is rank r's fp32 gradient of layer l (numpy).  Returns the
    scale exponents f~, each rank's packed codes, the reduced packed codes
    every rank ends with, and the unscaled/averaged fp32 outputs.
    ``n_threads`` splits the element loops over threads (bit-identical results).
    """
    p = len(grads)
    nl = len(grads[0])
    numels = np.array([np.asarray(g).size for g in grads[0]], dtype=np.int64)
    flat = [np.ascontiguousarray(grads[r][l], dtype=np.float32) for r in range(p) for l in range(nl)]
    gptrs = (ctypes.c_void_p * len(flat))(*[a.ctypes.data for a in flat])
    nbytes = packed_bytes(p, e, m, numels)
    ft = np.zeros(nl, dtype=np.int32)
    packed = np.zeros((p, nbytes), dtype=np.uint8) if want_packed else None
    reduced = np.zeros(nbytes, dtype=np.uint8)
    outs = [np.empty(int(n), dtype=np.float32) for n in numels] if want_out else None
    optrs = (ctypes.c_void_p * nl)(*[a.ctypes.data for a in outs]) if want_out else None
    rc = lib().oracle_aps_sync(p, e, m, nl, _ptr(numels), gptrs, average, _ptr(ft),
                               _ptr(packed) if want_packed else None, _ptr(reduced),
                               optrs, int(n_threads))
    return SyncResult(rc, ft, packed, reduced, outs)


def packed_bytes_mixed(p: int, numels, fmts) -> int:
    n = np.ascontiguousarray(numels, dtype=np.int64)
    e = np.ascontiguousarray([f[0] for f in fmts], dtype=np.int32)
    m = np.ascontiguousarray([f[1] for f in fmts], dtype=np.int32)
    return lib().oracle_packed_bytes_mixed(p, n.size, _ptr(n), _ptr(e), _ptr(m))


def aps_sync_mixed(grads, fmts, average: int = 1, want_packed: bool = True) -> SyncResult:
    """APS sync with per-layer formats fmts[l] = (e, m) (hybrid precision)."""
    p = len(grads)
    nl = len(grads[0])
    numels = np.array([np.asarray(g).size for g in grads[0]], dtype=np.int64)
    e = np.ascontiguousarray([f[0] for f in fmts], dtype=np.int32)
    m = np.ascontiguousarray([f[1] for f in fmts], dtype=np.int32)
    flat = [np.ascontiguousarray(grads[r][l], dtype=np.float32) for r in range(p) for l in range(nl)]
    gptrs = (ctypes.c_void_p * len(flat))(*[a.ctypes.data for a in flat])
    nbytes = packed_bytes_mixed(p, numels, fmts)
    ft = np.zeros(nl, dtype=np.int32)
    packed = np.zeros((p, nbytes), dtype=np.uint8) if want_packed else None
    reduced = np.zeros(nbytes, dtype=np.uint8)
    outs = [np.empty(int(n), dtype=np.float32) for n in numels]
    optrs = (ctypes.c_void_p * nl)(*[a.ctypes.data for a in outs])
    rc = lib().oracle_aps_sync_mixed(p, _ptr(e), _ptr(m), nl, _ptr(numels), gptrs, average, _ptr(ft),
                                     _ptr(packed) if want_packed else None, _ptr(reduced), optrs)
    return SyncResult(rc, ft, packed, reduced, outs)


def aps_sync_ex(grads, e: int, m: int, average: int = 1, group_k: int = 1, acc=None, kahan: int = 0,
                want_packed: bool = True, sr: int = 0, seed: int = 0) -> SyncResult:
    """APS sync with a reduction order and accumulator:
    ``group_k`` = hierarchical group size (1 or p: the flat ring, reading A23),
    ``acc`` = accumulator format (default: the wire format), ``kahan`` =
    compensated accumulation (reading A24)."""
    p = len(grads)
    nl = len(grads[0])
    ae, am = acc if acc is not None else (e, m)
    numels = np.array([np.asarray(g).size for g in grads[0]], dtype=np.int64)
    flat = [np.ascontiguousarray(grads[r][l], dtype=np.float32) for r in range(p) for l in range(nl)]
    gptrs = (ctypes.c_void_p * len(flat))(*[a.ctypes.data for a in flat])
    nbytes = packed_bytes(p, e, m, numels)
    ft = np.zeros(nl, dtype=np.int32)
    packed = np.zeros((p, nbytes), dtype=np.uint8) if want_packed else None
    reduced = np.zeros(nbytes, dtype=np.uint8)
    outs = [np.empty(int(n), dtype=np.float32) for n in numels]
    optrs = (ctypes.c_void_p * nl)(*[a.ctypes.data for a in outs])
    rc = lib().oracle_aps_sync_ex(p, e, m, nl, _ptr(numels), gptrs, average, group_k, ae, am, kahan, sr, seed,
                                  _ptr(ft),
                                  _ptr(packed) if want_packed else None, _ptr(reduced), optrs)
    return SyncResult(rc, ft, packed, reduced, outs)


def reduce1(codes, tile: int, tiles: int, group_k: int, e: int, m: int, acc=None, kahan: int = 0) -> int:
    """One element's all-reduce: codes[r] = rank r's wire code, ``tile`` its tile, ``tiles`` = T'."""
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    ae, am = acc if acc is not None else (e, m)
    return lib().oracle_reduce1(_ptr(c), c.size, tile, tiles, group_k, e, m, ae, am, kahan)


def round_off_error(grad_h, grad_l):
    """Eq. (5), reading A25: mean of |(h - l) / h| over h != 0.
    Returns (error, count)."""
    h = np.ascontiguousarray(grad_h, dtype=np.float32)
    l_ = np.ascontiguousarray(grad_l, dtype=np.float32)
    cnt = ctypes.c_int64(0)
    err = lib().oracle_round_off_error(_ptr(h), _ptr(l_), h.size, ctypes.byref(cnt))
    return err, cnt.value


def census(g, s: int, e: int, m: int) -> tuple[int, int]:
    """(underflow, overflow) counts of Cast(g * 2^s) over nonzero finite g (NEXT-4)."""
    x = np.ascontiguousarray(g, dtype=np.float32)
    u, o = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = lib().oracle_census(_ptr(x), x.size, s, e, m, ctypes.byref(u), ctypes.byref(o))
    if rc:
        raise ValueError(f"oracle_census rc={rc}")
    return u.value, o.value


def splitmix64(seed: int, ctr: int) -> int:
    return lib().oracle_splitmix64(seed, ctr)


def cast_sr1(x: float, e: int, m: int, r: int) -> int:
    """Stochastic-rounding Cast of one fp32 with the 32-bit random number r (reading A26)."""
    return lib().oracle_cast_sr1(x, e, m, r)


def cast_sr(x, e: int, m: int, seed: int, phase: int = 0) -> np.ndarray:
    """Stochastic-rounding Cast with r_i = SplitMix64(seed, phase << 40 | i) >> 32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint32)
    rc = lib().oracle_cast_sr(_ptr(x), _ptr(out), x.size, e, m, seed, phase)
    if rc:
        raise ValueError(f"oracle_cast_sr rc={rc}")
    return out
