"""Pins for the oracle's stochastic rounding (SURVEY 8(f) NEXT-4, P:397-398,
reading A26).  CPU only.

Independent of the oracle's code:
* SplitMix64's published output sequence for seed 0;
* hand-worked neighbour / probability cases;
* unbiasedness over 10^5 draws;
* a re-derivation of the whole SR pipeline with torch's float8_e5m2 for the
  nearest value, code-space neighbours, Fractions for the probability and a
  Python SplitMix64 (itself pinned by the published vectors).
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

import synthetic
from test_oracle_aps import EMPTY, _find_max_exp_literal, _pack_little

M64 = (1 << 64) - 1


def _splitmix(seed, ctr):
    z = (seed + (ctr + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_splitmix64_published_vectors(orc):
    """SplitMix64 seeded with 0 yields 0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4,
    0x06c45d188009454f (the reference generator's first outputs)."""
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [orc.splitmix64(0, i) for i in range(3)] == want
    assert [_splitmix(0, i) for i in range(3)] == want
    rng = np.random.default_rng(5)
    for _ in range(100):
        s, c = int(rng.integers(0, 2 ** 63)), int(rng.integers(0, 2 ** 50))
        assert orc.splitmix64(s, c) == _splitmix(s, c)


def test_sr_hand_cases(orc):
    """(5,2): 1.0625 lies a quarter of the way from 1.0 (0x3C) to 1.25 (0x3D):
    up iff r < 2^30.  Representable values never move.  3 * 2^-18 lies 3/4 of
    the way from 0 to the smallest subnormal 2^-16 (0x01).  61440 is halfway
    between 57344 (0x7B) and 2^16, the stand-in for Inf (0x7C)."""
    assert orc.cast_sr1(1.0625, 5, 2, 0) == 0x3D
    assert orc.cast_sr1(1.0625, 5, 2, 2 ** 30 - 1) == 0x3D
    assert orc.cast_sr1(1.0625, 5, 2, 2 ** 30) == 0x3C
    assert orc.cast_sr1(-1.0625, 5, 2, 0) == 0xBD
    for r in (0, 2 ** 31, 2 ** 32 - 1):
        assert orc.cast_sr1(1.25, 5, 2, r) == 0x3D
        assert orc.cast_sr1(0.0, 5, 2, r) == 0x00
        assert orc.cast_sr1(-0.0, 5, 2, r) == 0x80
    x = np.float32(3 * 2.0 ** -18)
    assert orc.cast_sr1(x, 5, 2, 3 * 2 ** 30 - 1) == 0x01
    assert orc.cast_sr1(x, 5, 2, 3 * 2 ** 30) == 0x00
    assert orc.cast_sr1(61440.0, 5, 2, 2 ** 31 - 1) == 0x7C
    assert orc.cast_sr1(61440.0, 5, 2, 2 ** 31) == 0x7B
    assert orc.cast_sr1(70000.0, 5, 2, 2 ** 32 - 1) == 0x7C        # past 2^(bias+1): Inf
    # (3,0): 3 lies halfway between 2 (0x4) and 4 (0x5)
    assert orc.cast_sr1(3.0, 3, 0, 2 ** 31 - 1) == 0x5 and orc.cast_sr1(3.0, 3, 0, 2 ** 31) == 0x4


@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (3, 0), (5, 6)])
def test_sr_unbiased(orc, fmt):
    """the mean of SR(x) over >= 10^5 draws lies within 3 standard errors of x."""
    e, m = fmt
    rng = np.random.default_rng([synthetic.SEED, 94, e, m])
    for x in (rng.uniform(1, 2, 4).astype(np.float32)):
        codes = orc.cast_sr(np.full(100_000, x, np.float32), e, m, seed=int(rng.integers(0, 2 ** 63)))
        v = orc.decode(codes, e, m).astype(np.float64)
        assert len(np.unique(v)) <= 2
        se = v.std() / np.sqrt(v.size) + 1e-12
        assert abs(v.mean() - float(x)) < 3 * se + 1e-9, (x, v.mean(), se)


def test_sr_at_8_23_is_exact(orc):
    """(8,23): every fp32 is representable, SR never moves a value: the SR
    pipeline equals the RNE one (transparency)."""
    g = synthetic.make_grads([300, 7], 4)
    a = orc.aps_sync_ex(g, 8, 23, average=1, sr=1, seed=99)
    b = orc.aps_sync_ex(g, 8, 23, average=1)
    assert np.array_equal(a.reduced, b.reduced)


def test_sr_argument_errors(orc):
    g = synthetic.make_grads([10], 2)
    assert orc.aps_sync_ex(g, 5, 2, sr=1, kahan=1).rc == 1
    assert orc.aps_sync_ex(g, 5, 2, sr=1, acc=(5, 10)).rc == 1


# ---------------------------------------------------------------- independent SR pipeline (5,2)

def _e5m2(x):
    return torch.from_numpy(np.asarray(x, np.float32).reshape(-1)).to(torch.float8_e5m2).view(torch.uint8).numpy()


def _val(c):
    return float(torch.tensor([c], dtype=torch.uint8).view(torch.float8_e5m2).float().item())


def _sr_e5m2(x, r):
    """SR in (5,2) from torch's nearest code and its code-space neighbour."""
    x = np.float32(x)
    if x == 0:
        return int(_e5m2(x)[0])
    c = int(_e5m2(x)[0])
    v = _val(c)
    if v == float(x):
        return c
    ax, av = abs(Fraction(float(x))), abs(Fraction(v))
    sign = c & 0x80
    mag = c & 0x7F
    lo_mag, hi_mag = (mag, mag + 1) if av < ax else (mag - 1, mag)
    lo, hi = abs(Fraction(_val(lo_mag))), (abs(Fraction(_val(hi_mag))) if hi_mag < 0x7C else Fraction(2 ** 16))
    up = r < (ax - lo) / (hi - lo) * 2 ** 32
    return sign | (hi_mag if up else lo_mag)


@pytest.mark.parametrize("p,k", [(2, 1), (4, 1), (4, 2), (6, 3)])
def test_sr_pipeline_independent(orc, p, k):
    e, m, seed = 5, 2, 0x1234_5678_9ABC
    numels = [40, 130]
    grads = synthetic.make_grads(numels, p, seed=synthetic.SEED + p)
    res = orc.aps_sync_ex(grads, e, m, average=1, group_k=k, sr=1, seed=seed)
    bias, G = 15, p // k
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
            for i in range(n):
                q[r, off + i] = _sr_e5m2(y[i], _splitmix(seed, (r << 40) | (off + i)) >> 32)
            off += 128 * ((n + 127) // 128)
    assert np.array_equal(res.packed, np.stack([_pack_little(q[r], 8) for r in range(p)]))
    s = np.zeros(Tp * 128, np.uint32)
    for i in range(Tp * 128):
        t = i // 128
        c1, c2 = t // (Tp // k), t // (Tp // G)
        a = 0
        S = None
        for gi in range(G):
            g = (c2 + 1 + gi) % G
            acc = _val(int(q[g * k + (c1 + 1) % k, i]))
            for j in range(1, k):
                a += 1
                x = np.float32(np.float32(acc) + np.float32(_val(int(q[g * k + (c1 + 1 + j) % k, i]))))
                acc = _val(_sr_e5m2(x, _splitmix(seed, ((p - 1 + a) << 40) | i) >> 32))
            if S is None:
                S = acc
            else:
                a += 1
                x = np.float32(np.float32(S) + np.float32(acc))
                S = _val(_sr_e5m2(x, _splitmix(seed, ((p - 1 + a) << 40) | i) >> 32))
        s[i] = _e5m2(S)[0]
    assert np.array_equal(res.reduced, _pack_little(s, 8))
