"""Pins for the oracle's reduction order (hierarchical all-reduce, SURVEY 8(f)
NEXT-3, reading A23), accumulator variants (CPD, NEXT-4, reading A24) and the
round-off metric (Eq. 5, reading A25).  CPU only.

Independent arithmetic used here (never the oracle's own code):
* hand-derived sums for all-equal inputs (the large-plus-small round-off the
  paper describes at P:531-537), worked out in the docstrings;
* torch float8_e5m2 / float16 / bfloat16 / float32 casts for the whole
  pipeline in the hierarchical order, with a wider accumulator, and with
  Kahan compensation;
* numpy float32 sums in the hierarchical order for (8,23) (transparency);
* exact Fractions for Eq. (5).
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

import synthetic
from test_oracle_aps import EMPTY, TORCH_DT, _find_max_exp_literal, _pack_little, _torch_codes, _torch_values

ACC_DT = {(5, 2): torch.float8_e5m2, (5, 10): torch.float16, (8, 7): torch.bfloat16, (8, 23): torch.float32,
          (4, 3): torch.float8_e4m3fn}


def _q(x, dt):
    """fp32 -> nearest value of dt (RNE), back as fp32 (library casts)."""
    x = np.ascontiguousarray(x, np.float32)
    if dt == torch.float32:
        return x.copy()
    return torch.from_numpy(x).to(dt).float().numpy()


# ---------------------------------------------------------------- hand-derived sums

def _all_equal(p, value=1.0):
    return [[np.array([value], np.float32)] for _ in range(p)]


@pytest.mark.parametrize("k, avg_out", [(1, 0.5), (2, 1.0), (4, 1.0), (8, 1.0), (16, 0.5)])
def test_hierarchical_all_equal_16_ranks(orc, k, avg_out):
    """p = 16 ranks each hold [1.0] under (5,2): A = 1, E = ceil(log2 16) = 4,
    f~ = 15 - 4 = 11, every scaled value v = 2048.  In (5,2) the binade
    [16384, 32768) has quantum 4096, so the flat ring (k = 1 or k = 16 = p)
    stagnates at 8v = 16384: 16384 + 2048 = 18432 is a tie between 16384 (even
    code) and 20480 -> 16384 ("add a local gradient with the
    summation of all other nodes' local gradients").  Groups of k = 8: each
    group sum stops exactly at 8v = 16384 (no tie is reached), two groups give
    32768 = 16v exactly.  k = 4: group sums 4v = 8192, then 16384, 24576,
    32768, all representable.  k = 2: group sums 4096, then 4096 * j for
    j = 1..8, all representable.  Average = sum / 2^11 / 16."""
    res = orc.aps_sync_ex(_all_equal(16), 5, 2, average=1, group_k=k)
    assert res.rc == 0 and res.ftilde[0] == 11
    assert res.out[0][0] == np.float32(avg_out)


def test_kahan_all_equal_16_ranks(orc):
    """Flat ring, 16 x v (v = 2048) in (5,2) with Kahan compensation:
    after 8v the plain sum stagnates; Kahan carries the lost v in c:
    9th: y = v, t = 8v (tie), c = (8v - 8v) - v = -v; 10th: y = 2v, t = 10v,
    c = 0; 11th: t = 11v -> 12v (tie to even), c = 2v - v = v; 12th: y = 0,
    t = 12v, c = 0; 13th: t = 13v -> 12v (tie), c = -v; 14th: y = 2v, t = 14v,
    c = 0; 15th: t = 15v -> 16v (tie), c = 2v - v = v; 16th: y = 0, t = 16v.
    The exact sum 16v = 32768: average 1.0."""
    res = orc.aps_sync_ex(_all_equal(16), 5, 2, average=1, group_k=1, kahan=1)
    assert res.out[0][0] == np.float32(1.0)
    plain = orc.aps_sync_ex(_all_equal(16), 5, 2, average=1, group_k=1, kahan=0)
    assert plain.out[0][0] == np.float32(0.5)


@pytest.mark.parametrize("acc", [(5, 10), (8, 7), (8, 23), (5, 6)])
def test_wide_accumulator_all_equal(orc, acc):
    """With any accumulator holding 3+ mantissa bits, j * v for j <= 16 is
    exact (j <= 16 needs 4 significant bits at most, and 16v = 2^15 <= the
    range of each format), so the sum is exact: average 1.0 ("we can use
    a higher precision to store the accumulator")."""
    res = orc.aps_sync_ex(_all_equal(16), 5, 2, average=1, group_k=1, acc=acc)
    assert res.out[0][0] == np.float32(1.0)


def test_three_rank_order_under_hierarchy(orc):
    """The order-sensitive input of test_ring_order_sensitivity (p = 3) lifted
    to p = 6 with groups of k = 3: ranks 0..2 hold [1.0], [0.125], [0.125] and
    ranks 3..5 hold zeros.  A = 1, E = ceil(log2 6) = 3, f~ = 12: scaled values
    4096, 512, 512.  One tile, T' = 6: chunk of group 0 is c1 = 0 (order 1, 2,
    0): 512 + 512 = 1024, + 4096 = 5120 (representable: 1.25 * 2^12) -> group
    sum 5120; group 1 sum = 0; masters chunk c2 = 0 over G = 2 groups: order
    1, 0: 0 + 5120 = 5120.  Sum 5120 / 2^12 = 1.25."""
    g = [[np.array([1.0], np.float32)], [np.array([0.125], np.float32)], [np.array([0.125], np.float32)]]
    g += [[np.array([0.0], np.float32)] for _ in range(3)]
    res = orc.aps_sync_ex(g, 5, 2, average=0, group_k=3)
    assert res.ftilde[0] == 12 and res.out[0][0] == np.float32(1.25)
    # flat ring over 6: chunk 0 order 1,2,3,4,5,0: 512+512 = 1024, +0+0+0, +4096 = 5120 as well
    # while the reversed hierarchy (rank 0 first) would round 4096 + 512 = 4608 -> 4096 (tie, even)
    c = orc.cast(np.array([4096.0, 512.0], np.float32), 5, 2)
    assert orc.ring_add(orc.ring_add(int(c[0]), int(c[1]), 5, 2), int(c[1]), 5, 2) == int(orc.cast(
        np.array([4096.0], np.float32), 5, 2)[0])


# ---------------------------------------------------------------- consistency with the flat oracle

@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 6)])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_flat_orders_equal_ring_oracle(orc, fmt, p):
    """k = 1 and k = p are the flat ring (A23); the accumulator equal to the
    wire format without compensation is O8 (A24)."""
    e, m = fmt
    numels = [5, 128, 300, 1, 1000]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 31 * p)
    ref = orc.aps_sync(grads, e, m, average=1)
    for k in sorted({1, p}):
        res = orc.aps_sync_ex(grads, e, m, average=1, group_k=k)
        assert res.rc == 0
        assert np.array_equal(res.ftilde, ref.ftilde)
        assert np.array_equal(res.packed, ref.packed)
        assert np.array_equal(res.reduced, ref.reduced)
        for a, b in zip(res.out, ref.out):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_ex_argument_errors(orc):
    g = synthetic.make_grads([10], 4)
    assert orc.aps_sync_ex(g, 5, 2, group_k=3).rc == 1      # k must divide p
    assert orc.aps_sync_ex(g, 5, 2, group_k=0).rc == 1
    assert orc.aps_sync_ex(g, 5, 2, acc=(1, 2)).rc == 2     # invalid accumulator format


# ---------------------------------------------------------------- independent re-derivation (torch casts)

def _independent_ex(grads, e, m, k, acc, kahan, average):
    """Alg. 1 with the reduction of readings A23/A24 re-derived with library
    casts: wire codes by a torch dtype, group folds over members in ring
    order c1+1..c1 of the group chunk, then over groups in ring order
    c2+1..c2 of the master chunk, each fp32 operation rounded by the
    accumulator's torch dtype."""
    dt, adt = TORCH_DT[(e, m)], ACC_DT[acc]
    bias = (1 << (e - 1)) - 1
    p = len(grads)
    G = p // k
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
            q[r, off:off + n] = _torch_codes(np.ldexp(grads[r][l].astype(np.float32), np.int32(ft[l])), dt)
            off += 128 * ((n + 127) // 128)
    vals = np.stack([_torch_values(q[r], dt) for r in range(p)]).astype(np.float32)   # [p, codes]
    tile = np.arange(Tp * 128) // 128
    c1 = tile // (Tp // k)
    c2 = tile // (Tp // G)
    idx = np.arange(Tp * 128)

    def fold(xs):
        s = _q(xs[0], adt)
        c = np.zeros_like(s)
        for x in xs[1:]:
            if not kahan:
                s = _q((s + x).astype(np.float32), adt)
            else:
                y = _q((x - c).astype(np.float32), adt)
                t = _q((s + y).astype(np.float32), adt)
                c = _q((_q((t - s).astype(np.float32), adt) - y).astype(np.float32), adt)
                s = t
        return s

    group_sums = []
    for gi in range(G):
        g = (c2 + 1 + gi) % G
        members = [vals[g * k + (c1 + 1 + j) % k, idx] for j in range(k)]
        group_sums.append(fold(members))
    S = fold(group_sums)
    s = _torch_codes(S, dt)
    outs, off = [], 0
    for l, n in enumerate(numels):
        v = _torch_values(s[off:off + n], dt)
        t = np.ldexp(v.astype(np.float32), np.int32(-ft[l]))
        if average:
            t = (t / np.float32(p)).astype(np.float32)
        outs.append(t)
        off += 128 * ((n + 127) // 128)
    return np.array(ft, np.int32), _pack_little(s, 1 + e + m), outs


CASES = [  # (fmt, p, k, acc, kahan)
    ((5, 2), 4, 2, (5, 2), 0), ((5, 2), 8, 2, (5, 2), 0), ((5, 2), 8, 4, (5, 2), 0), ((5, 2), 6, 3, (5, 2), 0),
    ((5, 2), 6, 2, (5, 2), 0), ((5, 2), 16, 4, (5, 2), 0), ((4, 3), 8, 4, (4, 3), 0),
    ((5, 2), 8, 1, (5, 10), 0), ((5, 2), 8, 1, (8, 23), 0), ((5, 2), 8, 4, (8, 7), 0), ((4, 3), 4, 1, (5, 10), 0),
    ((5, 2), 8, 1, (5, 2), 1), ((5, 2), 8, 2, (5, 2), 1), ((4, 3), 6, 3, (4, 3), 1), ((5, 2), 8, 1, (5, 10), 1),
    ((5, 10), 8, 2, (5, 10), 0), ((8, 7), 4, 2, (8, 7), 1),
]


@pytest.mark.parametrize("fmt, p, k, acc, kahan", CASES)
def test_ex_vs_torch_dtypes(orc, fmt, p, k, acc, kahan):
    e, m = fmt
    numels = [5, 128, 300, 1, 700]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + 7 * p + k)
    res = orc.aps_sync_ex(grads, e, m, average=1, group_k=k, acc=acc, kahan=kahan)
    ft, reduced, outs = _independent_ex(grads, e, m, k, acc, kahan, 1)
    assert res.rc == 0
    assert np.array_equal(res.ftilde, ft)
    assert np.array_equal(res.reduced, reduced)
    for a, b in zip(res.out, outs):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("p, k", [(4, 2), (8, 2), (8, 4), (6, 3), (12, 4)])
def test_hierarchical_transparency_8_23(orc, p, k):
    """(8,23): every re-quantise is the identity on fp32, so the result is the
    plain fp32 sum in the hierarchical order (S:269 transparency, A23)."""
    rng = np.random.default_rng([synthetic.SEED, 923, p, k])
    numels = [7, 129, 256, 1]
    grads = [[(rng.standard_normal(n) * 2.0 ** rng.integers(-20, 20)).astype(np.float32) for n in numels]
             for _ in range(p)]
    res = orc.aps_sync_ex(grads, 8, 23, average=0, group_k=k)
    T = sum((n + 127) // 128 for n in numels)
    Tp = p * ((T + p - 1) // p)
    flat = np.zeros((p, Tp * 128), np.float32)
    for r in range(p):
        off = 0
        for l, n in enumerate(numels):
            flat[r, off:off + n] = grads[r][l]
            off += 128 * ((n + 127) // 128)
    G = p // k
    ref = np.zeros(Tp * 128, np.float32)
    for i in range(Tp * 128):
        t = i // 128
        c1, c2 = t // (Tp // k), t // (Tp // G)
        S = None
        for gi in range(G):
            g = (c2 + 1 + gi) % G
            s = None
            for j in range(k):
                x = flat[g * k + (c1 + 1 + j) % k, i]
                s = x if s is None else np.float32(s + x)
            S = s if S is None else np.float32(S + s)
        ref[i] = S
    off = 0
    for l, n in enumerate(numels):
        assert np.array_equal(res.out[l], ref[off:off + n])
        off += 128 * ((n + 127) // 128)


# ---------------------------------------------------------------- Eq. (5)

def test_round_off_error_hand(orc):
    """Eq. (5): h = [1, 2, 0, 4], l = [1, 1, 5, 5]: terms 0, 1/2, (undefined,
    A25), 1/4 -> (0 + 0.5 + 0.25) / 3 = 0.25."""
    err, cnt = orc.round_off_error(np.array([1, 2, 0, 4], np.float32), np.array([1, 1, 5, 5], np.float32))
    assert cnt == 3 and err == 0.25
    err, cnt = orc.round_off_error(np.zeros(3, np.float32), np.ones(3, np.float32))
    assert cnt == 0 and err == 0.0


def test_round_off_error_vs_fractions(orc):
    rng = np.random.default_rng([synthetic.SEED, 595])
    h = (rng.standard_normal(2000) * 2.0 ** rng.integers(-30, 10, 2000)).astype(np.float32)
    h[::17] = 0.0
    l_ = (h * (1 + rng.standard_normal(2000) * 0.1)).astype(np.float32)
    err, cnt = orc.round_off_error(h, l_)
    terms = [abs((Fraction(float(a)) - Fraction(float(b))) / Fraction(float(a))) for a, b in zip(h, l_) if a != 0]
    exact = sum(terms) / len(terms)
    assert cnt == len(terms)
    assert abs(Fraction(err) - exact) <= exact * Fraction(1, 10 ** 12)


def test_round_off_error_hierarchy_beats_ring(orc):
    """the hierarchical all-reduce lowers Eq. (5) against the flat
    ring when many equal-magnitude gradients are summed.  All-equal input at
    p = 16 (test_hierarchical_all_equal_16_ranks): ring error 50 %, k = 4: 0."""
    g = _all_equal(16)
    h = np.array([1.0], np.float32)
    ring = orc.aps_sync_ex(g, 5, 2, average=1, group_k=1).out[0]
    hier = orc.aps_sync_ex(g, 5, 2, average=1, group_k=4).out[0]
    assert orc.round_off_error(h, ring)[0] == 0.5
    assert orc.round_off_error(h, hier)[0] == 0.0


# ---------------------------------------------------------------- underflow / overflow census (NEXT-4)

def test_census_fig_aps_comparing(orc):
    """Fig. `aps_comparing`, (5,2): a "green" layer with max 2^20 and a
    "blue" layer whose values sit near 2^-12.  No scaling: 2^20 > 61440 overflows
    (Inf).  Loss scaling by 2^-5 (the paper's constant): 2^20 -> 2^15 fits,
    but 2^-12 -> 2^-17 is the tie between 0 and 2^-16 and rounds to 0 (underflow,
    "smaller than 2^-16 ... cast to 0").  APS (N = 1): the green layer gets
    f~ = 15 - 20 = -5, the blue one (max 2^5 -> E = 5) f~ = 10: nothing lost."""
    green = np.array([2.0 ** 20, 1.0], np.float32)
    blue = np.array([2.0 ** 5, 2.0 ** -12, -(2.0 ** -12)], np.float32)
    assert orc.census(green, 0, 5, 2) == (0, 1)
    assert orc.census(blue, 0, 5, 2) == (0, 0)          # 2^-12 is a (5,2) subnormal: kept
    assert orc.census(green, -5, 5, 2) == (0, 0)
    assert orc.census(blue, -5, 5, 2) == (2, 0)
    fg = orc.scale_exp(5, orc.find_max_exp(green, 1))
    fb = orc.scale_exp(5, orc.find_max_exp(blue, 1))
    assert (fg, fb) == (-5, 10)
    assert orc.census(green, fg, 5, 2) == (0, 0) and orc.census(blue, fb, 5, 2) == (0, 0)


def test_census_thresholds(orc):
    """Exact thresholds from O6 (A10/A11): (5,2) 2^-17 -> 0 (tie to even code 0),
    nextafter(2^-17, inf) -> 2^-16; 61440 -> Inf (tie), 61439.99 -> 57344;
    zeros and non-finite inputs are not counted."""
    x = np.array([2.0 ** -17, np.nextafter(np.float32(2.0 ** -17), np.float32(1)), 61440.0, 61439.99,
                  0.0, -0.0, np.inf, np.nan, -(2.0 ** -17), -61440.0], np.float32)
    assert orc.census(x, 0, 5, 2) == (2, 2)


def test_census_aps_never_overflows(orc):
    """Eq. (1)-(4): with f~ from FindMaxExp the cast never overflows, for any N
    (section 3.3.2: APS trades the overflow side away completely)."""
    rng = np.random.default_rng([synthetic.SEED, 33])
    for (e, m) in [(5, 2), (4, 3), (3, 0), (5, 10)]:
        for N in (1, 2, 8, 256):
            g = (rng.standard_normal(5000) * 2.0 ** rng.integers(-40, 40)).astype(np.float32)
            f = orc.scale_exp(e, orc.find_max_exp(g, N))
            assert orc.census(g, f, e, m)[1] == 0
            # A * 2^f~ > 2^(bias-1) / N (maximality): log2(N) + 2 binades more and the max overflows
            assert orc.census(g, f + 2 + int(np.log2(N)), e, m)[1] > 0
