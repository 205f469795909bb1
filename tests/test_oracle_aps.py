"""Pins for oracle O2-O11 (FindMaxExp, f~, scale, ring sum, unscale, layout,
pack) against what the paper and the mathematics fix.  CPU only.

Independent arithmetic used here (never the oracle's own code):
* Python integers / fractions for ceil(log2(N |g|)) (Alg. 1 FindMaxExp);
* torch's float8_e5m2 / float16 / bfloat16 / float8_e4m3fn casts for the whole
  pipeline of Alg. 1 in the formats that equal a torch dtype;
* numpy.packbits(bitorder="little") for the O11 bit layout;
* brute-force nearest-value search over Fractions for the ring add (A13).
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import synthetic

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EMPTY = -(2 ** 31)


# ---------------------------------------------------------------- FindMaxExp

def _ceil_log2_fraction(q: Fraction) -> int:
    """smallest integer E with 2^E >= q (q > 0), by integer arithmetic."""
    E = q.numerator.bit_length() - q.denominator.bit_length() - 1
    while Fraction(2) ** E < q:
        E += 1
    while Fraction(2) ** (E - 1) >= q:
        E -= 1
    return E


def _find_max_exp_literal(g, N):
    """Alg. 1 FindMaxExp(g * N), literally: max over i != 0 of
    ceil(log2(abs(i))) with exact arithmetic; -INF for an all-zero tensor."""
    mx = EMPTY
    for x in g:
        x = float(x)
        if x != 0.0:
            mx = max(mx, _ceil_log2_fraction(abs(Fraction(x)) * N))
    return mx


def test_find_max_exp_spec_examples(orc):
    """[0.75, -0.5, 0.0] -> 0; [2.0] -> 1; [0, 0] -> Empty."""
    assert orc.find_max_exp(np.array([0.75, -0.5, 0.0], np.float32), 1) == 0
    assert orc.find_max_exp(np.array([2.0], np.float32), 1) == 1
    assert orc.find_max_exp(np.array([0.0, -0.0], np.float32), 1) == EMPTY
    assert orc.find_max_exp(np.array([np.inf], np.float32), 1) == 2 ** 31 - 1


def test_find_max_exp_literal_alg1(orc):
    rng = np.random.default_rng([synthetic.SEED, 11])
    for trial in range(300):
        n = int(rng.integers(1, 40))
        bits = rng.integers(0, 0x7F800000, n).astype(np.uint32)
        if trial % 3 == 0:
            bits = bits % np.uint32(1 << 23)                   # fp32 subnormals (A5)
        if trial % 5 == 0:
            bits = (rng.integers(1, 254, n).astype(np.uint32) << np.uint32(23))  # exact powers of 2
        g = (bits | (rng.integers(0, 2, n).astype(np.uint32) << np.uint32(31))).view(np.float32)
        g[rng.random(n) < 0.2] = 0.0
        N = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 12, 100, 256]))
        assert orc.find_max_exp(g, N) == _find_max_exp_literal(g, N), (g, N)


# ---------------------------------------------------------------- f~ and Eq. (1)-(4)

def _golden_rows(kind):
    with open(os.path.join(GOLDEN, "paper_examples.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if line and line[0] == kind:
                yield line[1:]


def test_paper_aps_shifts(orc):
    """under (5,2) APS scales the blue layer by 2^10 and the green layer
    by 2^-5 (golden rows aps_shift)."""
    rows = list(_golden_rows("aps_shift"))
    assert len(rows) >= 4
    for e, m, N, amax, ft in rows:
        e, m, N, amax, ft = int(e), int(m), int(N), float(amax), int(ft)
        layer = np.array([amax * 0.25, -amax, 0.0, amax / 3], np.float32)
        res = orc.aps_sync([[layer]] * N, e, m, average=1)
        assert res.rc == 0
        assert res.ftilde[0] == ft


def test_spec_scale_exponent_example(orc):
    """(5,2), max exponent -20 with N = 256 -> f~ = 15 - (-12) = 27."""
    assert orc.scale_exp(5, -12) == 27
    assert orc.scale_exp(5, 15) == 0
    assert orc.scale_exp(5, EMPTY) == 0             # all-zero layer (A3)


@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10), (8, 7), (2, 1)])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 8, 16])
def test_eq4_bound_and_maximality(orc, fmt, N):
    """Eq. (3): f <= p^ / |N g^|, p^ = 2^upper_bound_exp (A1); Eq. (4)
    P:375 picks the largest power of two, so f~ + 1 breaks the bound."""
    e, m = fmt
    bias = orc.bias(e)
    rng = np.random.default_rng([synthetic.SEED, e, m, N])
    for _ in range(20):
        grads = [[(rng.standard_normal(37) * 2.0 ** rng.integers(-30, 30)).astype(np.float32)]
                 for _ in range(N)]
        res = orc.aps_sync(grads, e, m, want_packed=False, want_out=False)
        ghat = max(float(np.max(np.abs(g[0]))) for g in grads)
        ft = int(res.ftilde[0])
        bound = Fraction(2) ** bias
        assert Fraction(2) ** ft * N * Fraction(ghat) <= bound
        assert Fraction(2) ** (ft + 1) * N * Fraction(ghat) > bound


@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10)])
@pytest.mark.parametrize("N", [2, 3, 16, 256])
def test_no_overflow_adversarial(orc, fmt, N):
    """Section 3.3.2 / Eq. (1): with APS no partial sum overflows;
    adversarial all-equal max-magnitude inputs: zero Inf."""
    e, m = fmt
    vals = np.array([1.0, 0.75, 1.0 - 2.0 ** -20, 3.0, 1.5 * 2 ** -9], np.float32)
    for v in vals:
        layer = np.full(130, v, np.float32)
        layer[::7] = -v if N > 2 else v
        grads = [[layer] for _ in range(N)]
        res = orc.aps_sync(grads, e, m, average=0, want_packed=False)
        assert res.rc == 0
        assert np.all(np.isfinite(res.out[0]))
        b = 1 + e + m
        codes = np.array([int(c) for c in _unpack_little(res.reduced, b)], np.uint32)
        assert not np.any(((codes >> m) & ((1 << e) - 1)) == (1 << e) - 1)   # no Inf/NaN code


# ---------------------------------------------------------------- layout / pack

def _unpack_little(buf, b):
    bits = np.unpackbits(np.asarray(buf, np.uint8), bitorder="little")
    n = bits.size // b
    bits = bits[: n * b].reshape(n, b).astype(np.uint64)
    return (bits << np.arange(b, dtype=np.uint64)).sum(axis=1).astype(np.uint32)


def _pack_little(codes, b):
    c = np.asarray(codes, np.uint64)
    bits = ((c[:, None] >> np.arange(b, dtype=np.uint64)) & 1).astype(np.uint8).ravel()
    return np.packbits(bits, bitorder="little")


@pytest.mark.parametrize("b", [3, 4, 5, 7, 8, 9, 12, 16, 17, 24, 31, 32])
def test_pack_vs_numpy_packbits(orc, b):
    """O11: code i at bits [i b, (i+1) b), LSB-first -- numpy.packbits is an
    independent implementation of that layout."""
    rng = np.random.default_rng([synthetic.SEED, b])
    n = 128 * 5 + 3
    codes = rng.integers(0, 2 ** b, n, dtype=np.uint64).astype(np.uint32)
    ours = orc.pack(codes, b)
    assert np.array_equal(ours, _pack_little(codes, b))
    assert np.array_equal(orc.unpack(ours, n, b), codes)


def test_pack_hand_bytes(orc):
    """(5,2) [1.0, -2.0] -> bytes 3C C0 ("0b0_01111_00" = 0x3C for 1.0);
    (3,0) [1.0, -2.0] -> codes 0x3, 0xC -> one LSB-first byte 0xC3 (A17)."""
    c = orc.cast(np.array([1.0, -2.0], np.float32), 5, 2)
    assert list(orc.pack(c, 8)) == [0x3C, 0xC0]
    c = orc.cast(np.array([1.0, -2.0], np.float32), 3, 0)
    assert list(c) == [0x3, 0xC]
    assert list(orc.pack(c, 4)) == [0xC3]


def test_layout_tiles(orc):
    """O7: T_l = ceil(n_l/128), T' = p ceil(T/p); packed bytes = 16 b T'."""
    numels = synthetic.RESNET50_NUMELS
    T = sum((n + 127) // 128 for n in numels)
    assert T == 199_672
    for p in (1, 2, 3, 4, 7, 8):
        Tp = orc.total_tiles(p, numels)
        assert Tp % p == 0 and T <= Tp < T + p
        for e, m in [(5, 2), (3, 0), (5, 6), (5, 10)]:
            assert orc.packed_bytes(p, e, m, numels) == 16 * (1 + e + m) * Tp


# ---------------------------------------------------------------- whole pipeline via torch casts

TORCH_DT = {(5, 2): torch.float8_e5m2, (5, 10): torch.float16, (8, 7): torch.bfloat16,
            (4, 3): torch.float8_e4m3fn}


def _torch_codes(x32, dt):
    t = torch.from_numpy(np.ascontiguousarray(x32, np.float32)).to(dt)
    if t.element_size() == 1:
        return t.view(torch.uint8).numpy().astype(np.uint32)
    return t.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32)


def _torch_values(codes, dt):
    c = np.asarray(codes)
    if dt in (torch.float8_e5m2, torch.float8_e4m3fn):
        return torch.from_numpy(c.astype(np.uint8)).view(dt).float().numpy()
    return torch.from_numpy(c.astype(np.uint16).view(np.int16)).view(dt).float().numpy()


def _independent_aps(grads, e, m, average):
    """Alg. 1 re-derived with library casts: E by exact integer
    log2, scale by numpy float32 ldexp, Cast by a torch dtype, the ring
     with a fp32 add and re-cast after every add in the
    order of reading A14, cast back by torch, unscale by ldexp, average by a
    float32 division."""
    dt = TORCH_DT[(e, m)]
    bias = (1 << (e - 1)) - 1
    p = len(grads)
    numels = [g.size for g in grads[0]]
    ft = []
    for l in range(len(numels)):
        E = max(_find_max_exp_literal(grads[r][l], p) for r in range(p))
        ft.append(0 if E == EMPTY else bias - E)
    T = sum((n + 127) // 128 for n in numels)
    Tp = p * ((T + p - 1) // p)
    q = np.zeros((p, Tp * 128), np.uint32)
    for r in range(p):
        off = 0
        for l, n in enumerate(numels):
            y = np.ldexp(grads[r][l].astype(np.float32), np.int32(ft[l]))
            q[r, off:off + n] = _torch_codes(y, dt)
            off += 128 * ((n + 127) // 128)
    chunk = Tp // p * 128
    s = np.zeros(Tp * 128, np.uint32)
    for c in range(p):
        sl = slice(c * chunk, (c + 1) * chunk)
        acc = q[(c + 1) % p, sl]
        for j in range(2, p + 1):
            v = _torch_values(acc, dt) + _torch_values(q[(c + j) % p, sl], dt)   # fp32 add
            acc = _torch_codes(v.astype(np.float32), dt)
        s[sl] = acc
    outs, off = [], 0
    for l, n in enumerate(numels):
        v = _torch_values(s[off:off + n], dt)
        t = np.ldexp(v.astype(np.float32), np.int32(-ft[l]))
        if average:
            t = (t / np.float32(p)).astype(np.float32)
        outs.append(t)
        off += 128 * ((n + 127) // 128)
    b = 1 + e + m
    return (np.array(ft, np.int32), np.stack([_pack_little(q[r], b) for r in range(p)]),
            _pack_little(s, b), outs)


@pytest.mark.parametrize("fmt", list(TORCH_DT))
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_pipeline_vs_torch_dtypes(orc, fmt, p):
    e, m = fmt
    numels = [5, 128, 300, 1]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 17 * p)
    for average in (0, 1):
        res = orc.aps_sync(grads, e, m, average=average)
        ft, packed, reduced, outs = _independent_aps(grads, e, m, average)
        assert res.rc == 0
        assert np.array_equal(res.ftilde, ft)
        assert np.array_equal(res.packed, packed)
        assert np.array_equal(res.reduced, reduced)
        for a, b_ in zip(res.out, outs):
            assert np.array_equal(a.view(np.uint32), b_.view(np.uint32))


def test_worked_example_p2(orc):
    """p = 2, (5,2), one layer of four elements, average = 1 (SURVEY 8(c) worked
    example, re-derived independently by _independent_aps)."""
    r0 = np.array([0.75, -0.5, 0.0, 3e-6], np.float32)
    r1 = np.array([0.1, 0.25, -0.3, -0.0], np.float32)
    res = orc.aps_sync([[r0], [r1]], 5, 2, average=1)
    assert res.ftilde[0] == 14                              # A = 0.75, E = ceil(log2 1.5) = 1
    assert list(res.packed[0][:4]) == [0x72, 0xF0, 0x00, 0x2A]
    assert list(res.packed[1][:4]) == [0x66, 0x6C, 0xED, 0x80]
    assert list(res.reduced[:4]) == [0x73, 0xEC, 0xED, 0x2A]
    assert [hex(v) for v in res.out[0].view(np.uint32)] == \
        ["0x3ee00000", "0xbe000000", "0xbe200000", "0x35c00000"]
    ft, packed, reduced, outs = _independent_aps([[r0], [r1]], 5, 2, 1)
    assert np.array_equal(res.reduced, reduced) and np.array_equal(res.out[0], outs[0])


def test_ring_order_sensitivity(orc):
    """p = 3, (5,2), ranks hold [1.0], [0.125], [0.125]: A = 1, E = ceil(log2 3) = 2,
    f~ = 13, scaled values 8192, 1024, 1024.  Chunk 0 is accumulated in order
    1, 2, 0 (A14): 1024 + 1024 = 2048, + 8192 = 10240 = 1.25 * 2^13 -> 0x71.
    The order 0, 1, 2 would give 8192 + 1024 = 9216 (a tie -> 8192, even code),
    then 9216 -> 8192 again: 0x70.  So this input catches any order bug."""
    res = orc.aps_sync([[np.array([1.0], np.float32)], [np.array([0.125], np.float32)],
                        [np.array([0.125], np.float32)]], 5, 2, average=0)
    assert res.ftilde[0] == 13
    assert res.reduced[0] == 0x71
    assert res.out[0][0] == np.float32(1.25)
    # the wrong order, with the oracle's own add, gives 0x70
    c = orc.cast(np.array([8192.0, 1024.0], np.float32), 5, 2)
    assert orc.ring_add(orc.ring_add(int(c[0]), int(c[1]), 5, 2), int(c[1]), 5, 2) == 0x70


def test_stagnation_3_0(orc):
    """(3,0), p = 8, every rank [0.5]: N A = 4, E = 2, f~ = 3 - 2 = 1, each scaled
    value is 1.0; 1 + 1 = 2; 2 + 1 = 3 is a tie between 2 (code 0x4, even) and 4
    (0x5), so the sum stagnates at 2 (A9): the large-plus-small round-off of
    P:531-537.  Unscaled sum 1.0 instead of 4.0."""
    res = orc.aps_sync([[np.array([0.5], np.float32)]] * 8, 3, 0, average=0)
    assert res.ftilde[0] == 1
    assert res.reduced[0] & 0xF == 0x4
    assert res.out[0][0] == np.float32(1.0)


def test_transparency_8_23(orc):
    """S:269 / S:412: at (8,23) APS is the plain fp32 ring sum in the same
    order (power-of-two scaling is exact, section 3.3.1)."""
    rng = np.random.default_rng([synthetic.SEED, 823])
    for p in (1, 2, 3, 5, 8):
        numels = [7, 129, 256]
        grads = [[(rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20)).astype(np.float32)
                  for n in numels] for _ in range(p)]
        res = orc.aps_sync(grads, 8, 23, average=0)
        T = sum((n + 127) // 128 for n in numels)
        Tp = p * ((T + p - 1) // p)
        flat = np.zeros((p, Tp * 128), np.float32)
        for r in range(p):
            off = 0
            for l, n in enumerate(numels):
                flat[r, off:off + n] = grads[r][l]
                off += 128 * ((n + 127) // 128)
        chunk = Tp // p * 128
        ref = np.zeros(Tp * 128, np.float32)
        for c in range(p):
            sl = slice(c * chunk, (c + 1) * chunk)
            acc = flat[(c + 1) % p, sl].copy()
            for j in range(2, p + 1):
                acc = (acc + flat[(c + j) % p, sl]).astype(np.float32)
            ref[sl] = acc
        off = 0
        for l, n in enumerate(numels):
            assert np.array_equal(res.out[l], ref[off:off + n])
            off += 128 * ((n + 127) // 128)


def _rne_fraction(x: Fraction, e, m):
    """Exact nearest (e,m) value of a Fraction (ties -> even code), by search."""
    bias = (1 << (e - 1)) - 1
    vals = []
    for E in range(0, (1 << e) - 1):
        for M in range(1 << m):
            vals.append(Fraction(M, 2 ** (m + bias - 1)) if E == 0 else
                        Fraction((1 << m) + M) * Fraction(2) ** (E - bias - m))
    vals.append(Fraction(2) ** (bias + 1))          # Inf stand-in
    a = abs(x)
    best = min(range(len(vals)), key=lambda i: (abs(vals[i] - a), i % 2))
    code = best if best < len(vals) - 1 else ((1 << e) - 1) << m
    if a >= Fraction(2) ** (bias + 1):
        code = ((1 << e) - 1) << m
    return code | ((1 << (e + m)) if x < 0 else 0)


@pytest.mark.parametrize("fmt", [(3, 0), (2, 1), (4, 3), (5, 2)])
def test_ring_add_equals_exact_rounding(orc, fmt):
    """A13: cast(fl32(a + b)) equals one exact RNE of a + b for m <= 10
    (2p+1 double-rounding bound); checked on all (3,0)/(2,1) pairs and on
    sampled (4,3)/(5,2) pairs with exact Fractions."""
    e, m = fmt
    b = 1 + e + m
    n = 1 << b
    codes = [c for c in range(n) if ((c >> m) & ((1 << e) - 1)) != (1 << e) - 1]
    if n > 64:
        rng = np.random.default_rng([synthetic.SEED, e, m])
        pairs = [(int(rng.choice(codes)), int(rng.choice(codes))) for _ in range(1500)]
    else:
        pairs = [(a, c) for a in codes for c in codes]
    vals = orc.decode(np.arange(n, dtype=np.uint32), e, m)
    for a, c in pairs:
        exact = Fraction(float(vals[a])) + Fraction(float(vals[c]))
        if exact == 0:
            continue                          # signed-zero rule is IEEE (A15), tested elsewhere
        assert orc.ring_add(a, c, e, m) == _rne_fraction(exact, e, m), (hex(a), hex(c))


def test_underflow_rescue(orc):
    """Fig. `aps_comparing` mechanism, SPEC S:414 / S:271: a layer
    whose max exponent is far below 2^-(16+log2 N) underflows entirely in (5,2)
    without scaling (Eq. 5 error 1.0) but survives with APS."""
    N = 8
    rng = np.random.default_rng([synthetic.SEED, 414])
    grads = [[np.abs(rng.lognormal(-10, 2, 4096)).astype(np.float32) * np.float32(2.0 ** -30)]
             for _ in range(N)]
    ref = np.sum(np.stack([g[0].astype(np.float64) for g in grads]), axis=0) / N
    # no scaling: cast, then ring sum (f~ = 0 policy)
    q = [orc.cast(g[0], 5, 2) for g in grads]
    assert all(np.all(orc.decode(c, 5, 2) == 0) for c in q)
    err_noscale = np.mean(np.abs((ref - 0.0) / ref))           # Eq. (5)
    res = orc.aps_sync(grads, 5, 2, average=1)
    err_aps = np.mean(np.abs((ref - res.out[0]) / ref))
    assert err_noscale == 1.0
    assert err_aps < 0.5


def test_nonfinite_reported(orc):
    g = [[np.array([1.0, np.nan], np.float32)], [np.array([1.0, 2.0], np.float32)]]
    assert orc.aps_sync(g, 5, 2).rc == 6
    g = [[np.array([1.0, np.inf], np.float32)]]
    assert orc.aps_sync(g, 5, 2).rc == 6


def test_all_zero_layer(orc):
    """A3: an all-zero layer gets f~ = 0 and its (signed) zeros are transmitted."""
    g = [[np.array([0.0, -0.0, 0.0], np.float32), np.array([1.0], np.float32)],
         [np.array([-0.0, -0.0, 0.0], np.float32), np.array([1.0], np.float32)]]
    res = orc.aps_sync(g, 5, 2, average=1)
    assert res.ftilde[0] == 0
    assert [hex(v) for v in res.out[0].view(np.uint32)] == ["0x0", "0x80000000", "0x0"]


# ---------------------------------------------------------------- per-layer formats (NEXT-2)

@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_mixed_uniform_equals_uniform(orc, p):
    """The per-layer-format oracle with one format everywhere is the uniform oracle."""
    numels = [5, 128, 300, 1, 1000]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 5)
    for fmt in [(5, 2), (3, 0), (5, 6)]:
        a = orc.aps_sync(grads, *fmt, average=1)
        b = orc.aps_sync_mixed(grads, [fmt] * len(numels), average=1)
        assert np.array_equal(a.ftilde, b.ftilde)
        assert np.array_equal(a.packed, b.packed) and np.array_equal(a.reduced, b.reduced)
        for x, y in zip(a.out, b.out):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def _independent_mixed(grads, fmts, average):
    """Hybrid precision re-derived per layer with library casts (torch dtypes;
    (8,23) = fp32 itself, section 3.3.1: power-of-two scaling is exact), the
    ring in the order of A14, and the per-tile packed layout written with
    numpy.packbits."""
    p = len(grads)
    numels = [g.size for g in grads[0]]
    T = sum((n + 127) // 128 for n in numels)
    Tp = p * ((T + p - 1) // p)
    lay = np.concatenate([np.full(128 * ((n + 127) // 128), l) for l, n in enumerate(numels)]
                         + [np.full(128 * (Tp - T), len(numels) - 1)])
    def codes_of(x, fmt):
        if fmt == (8, 23):
            return np.ascontiguousarray(x, np.float32).view(np.uint32).copy()
        return _torch_codes(x, TORCH_DT[fmt])
    def vals_of(c, fmt):
        if fmt == (8, 23):
            return np.ascontiguousarray(c, np.uint32).view(np.float32)
        return _torch_values(c, TORCH_DT[fmt])
    ft = []
    for l, fmt in enumerate(fmts):
        E = max(_find_max_exp_literal(grads[r][l], p) for r in range(p))
        ft.append(0 if E == EMPTY else ((1 << (fmt[0] - 1)) - 1) - E)
    q = np.zeros((p, Tp * 128), np.uint32)
    for r in range(p):
        off = 0
        for l, n in enumerate(numels):
            q[r, off:off + n] = codes_of(np.ldexp(grads[r][l], np.int32(ft[l])), fmts[l])
            off += 128 * ((n + 127) // 128)
    chunk = Tp // p * 128
    s = np.zeros(Tp * 128, np.uint32)
    for i0 in range(0, Tp * 128, 128):
        fmt = fmts[lay[i0]]
        c = i0 // chunk
        sl = slice(i0, i0 + 128)
        acc = q[(c + 1) % p, sl]
        for j in range(2, p + 1):
            v = (vals_of(acc, fmt) + vals_of(q[(c + j) % p, sl], fmt)).astype(np.float32)
            acc = codes_of(v, fmt)
        s[sl] = acc
    def pack(codes):
        parts = []
        for i0 in range(0, Tp * 128, 128):
            fmt = fmts[lay[i0]]
            parts.append(_pack_little(codes[i0:i0 + 128], 1 + fmt[0] + fmt[1]))
        return np.concatenate(parts)
    outs, off = [], 0
    for l, n in enumerate(numels):
        t = np.ldexp(vals_of(s[off:off + n], fmts[l]).astype(np.float32), np.int32(-ft[l]))
        outs.append((t / np.float32(p)).astype(np.float32) if average else t)
        off += 128 * ((n + 127) // 128)
    return np.array(ft, np.int32), np.stack([pack(q[r]) for r in range(p)]), pack(s), outs


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_mixed_hybrid_vs_torch(orc, p):
    """Hybrid precision: (5,2) everywhere, (8,23) = fp32 for the classifier
    weight and bias (Table `last_layer_precision`), plus a (5,10) layer."""
    numels = [300, 128, 4096, 1000, 1]
    fmts = [(5, 2), (5, 10), (5, 2), (8, 23), (8, 23)]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 9)
    res = orc.aps_sync_mixed(grads, fmts, average=1)
    ft, packed, reduced, outs = _independent_mixed(grads, fmts, 1)
    assert res.rc == 0
    assert np.array_equal(res.ftilde, ft)
    assert np.array_equal(res.packed, packed)
    assert np.array_equal(res.reduced, reduced)
    for a, b in zip(res.out, outs):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("p,fmt", [(1, (5, 2)), (3, (4, 3)), (4, (3, 0)), (8, (5, 6))])
def test_oracle_threads_bit_identical(orc, p, fmt):
    """The all-cores oracle (bench.py's cpu_baseline) splits only the element loops:
    f~, every rank's codes, the reduced codes and the outputs are bit-identical for
    any thread count (ranges cross layer and chunk boundaries: 600000 > OR_RANGE)."""
    e, m = fmt
    numels = synthetic.C1_NUMELS + [1000, 1, 9408, 130, 8195, 600000]
    grads = synthetic.make_grads(numels, p)
    one = orc.aps_sync(grads, e, m, n_threads=1)
    assert one.rc == 0
    for nt in (2, 5, 8):
        r = orc.aps_sync(grads, e, m, n_threads=nt)
        assert r.rc == 0
        assert np.array_equal(r.ftilde, one.ftilde)
        assert np.array_equal(r.packed, one.packed)
        assert np.array_equal(r.reduced, one.reduced)
        for a, b in zip(r.out, one.out):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    edge = synthetic.edge_case_layers(p)
    assert np.array_equal(orc.aps_sync(edge, e, m, n_threads=4).reduced, orc.aps_sync(edge, e, m).reduced)
