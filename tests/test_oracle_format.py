"""Pins for oracle O1 (format, decode) and O6 (cast) against what the paper
and independent libraries fix.  CPU only.

* Table `precision_range` -> tests/golden/table2_precision_range.txt
* P:277-278 / P:300 overflow / underflow statements -> tests/golden/paper_examples.txt
* torch's float8_e5m2 / float16 / bfloat16 / float8_e4m3fn conversions are
  independent implementations of (5,2) / (5,10) / (8,7) / (4,3) (the last only
  below 248, where OCP e4m3fn and IEEE-style (4,3) coincide; reading A12).
* brute-force argmin over every representable value of every format with
  b = 1+e+m <= 12 (plus sampled (5,10)): a different algorithm from the
  oracle's lo/hi bracketing.
"""
import math
import os

import numpy as np
import pytest
import torch

import synthetic

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- Table 2

@pytest.mark.parametrize("row", _golden("table2_precision_range.txt"), ids=lambda r: r[0])
def test_table2_ranges(orc, row):
    """Table `precision_range` P:190-194: range [2^lo, 2^hi] = (smallest positive
    subnormal, exponent of the largest finite value)."""
    _, e, m, lo, hi = row
    e, m, lo, hi = int(e), int(m), int(lo), int(hi)
    assert orc.format_valid(e, m)
    assert orc.decode([1], e, m)[0] == np.float32(2.0 ** lo)          # min subnormal code 0..01
    maxfinite_code = (((1 << e) - 2) << m) | ((1 << m) - 1)
    v = float(orc.decode([maxfinite_code], e, m)[0])
    assert 2.0 ** hi <= v < 2.0 ** (hi + 1)
    # the next code up is +Inf (IEEE-style reserved exponent, A12)
    assert math.isinf(orc.decode([maxfinite_code + 1], e, m)[0])
    assert orc.bias(e) == hi                                           # upper_bound_exp


def test_paper_examples_cast(orc):
    """(5,2) values > 2^15 overflow to INF, values below 2^-16 go to 0."""
    n = 0
    for row in _golden("paper_examples.txt"):
        kind = row[0]
        if kind == "overflow_to_inf":
            e, m, x = int(row[1]), int(row[2]), float(row[3])
            for s in (1.0, -1.0):
                v = orc.decode(orc.cast([s * x], e, m), e, m)[0]
                assert np.isinf(v) and np.sign(v) == s
            n += 1
        elif kind == "underflow_to_zero":
            e, m, x = int(row[1]), int(row[2]), float(row[3])
            for s in (1.0, -1.0):
                c = orc.cast([s * x], e, m)[0]
                assert orc.decode([c], e, m)[0] == 0.0
                assert c == (0 if s > 0 else 1 << (e + m))                 # signed zero (A15)
            n += 1
        elif kind == "upper_bound_exp":
            assert orc.bias(int(row[1])) == int(row[2])
            n += 1
    assert n >= 8


def test_format_validity(orc):
    assert not orc.format_valid(1, 2)       # e = 1: bias 0, no normals (reading A-format)
    assert not orc.format_valid(9, 2)
    assert not orc.format_valid(5, 24)
    assert not orc.format_valid(8, 24)      # 33 bits
    assert orc.format_valid(8, 23) and orc.format_valid(2, 0) and orc.format_valid(3, 0)


# ---------------------------------------------------------------- torch dtypes

TORCH_FORMATS = [
    ((5, 2), torch.float8_e5m2, torch.uint8, None),
    ((5, 10), torch.float16, torch.int16, None),
    ((8, 7), torch.bfloat16, torch.int16, None),
    ((4, 3), torch.float8_e4m3fn, torch.uint8, 248.0),
]


@pytest.mark.parametrize("fmt,dt,it,limit", TORCH_FORMATS, ids=lambda x: str(x))
def test_decode_all_codes_vs_torch(orc, fmt, dt, it, limit):
    e, m = fmt
    b = 1 + e + m
    codes = np.arange(1 << b, dtype=np.uint32)
    ours = orc.decode(codes, e, m)
    if it == torch.uint8:
        ref = torch.from_numpy(codes.astype(np.uint8)).view(dt).float().numpy()
    else:
        ref = torch.from_numpy(codes.astype(np.uint16).view(np.int16)).view(dt).float().numpy()
    if limit is not None:       # (4,3) vs OCP e4m3fn: only the codes below 248 coincide
        keep = np.abs(ref) < limit
        keep &= (codes & 0x7F) < 0x78
    else:
        keep = np.ones_like(ours, dtype=bool)
    both_nan = np.isnan(ours) & np.isnan(ref)
    sel = keep & ~both_nan
    assert np.array_equal(ours[sel].view(np.uint32), ref[sel].view(np.uint32))
    assert np.array_equal(np.isnan(ours[keep]), np.isnan(ref[keep]))


@pytest.mark.parametrize("fmt,dt,it,limit", TORCH_FORMATS, ids=lambda x: str(x))
def test_cast_vs_torch(orc, fmt, dt, it, limit):
    e, m = fmt
    x = synthetic.fp32_probe_patterns(1 << 21)
    # midpoints of neighbouring codes and +-1 ulp around them (rounding corners)
    b = 1 + e + m
    allc = np.arange(1 << min(b, 16), dtype=np.uint32)
    vals = orc.decode(allc, e, m).astype(np.float64)
    vals = np.unique(vals[np.isfinite(vals)])
    mids = ((vals[1:] + vals[:-1]) / 2).astype(np.float32)
    corners = np.concatenate([mids, np.nextafter(mids, np.float32(np.inf)),
                              np.nextafter(mids, np.float32(-np.inf)), vals.astype(np.float32)])
    x = np.concatenate([x, corners, -corners])
    x = x[~np.isnan(x)]
    if limit is not None:
        x = x[np.abs(x) < limit]
    ours = orc.cast(x, e, m)
    t = torch.from_numpy(x).to(dt)
    if it == torch.uint8:
        ref = t.view(torch.uint8).numpy().astype(np.uint32)
    else:
        ref = t.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32)
    bad = np.nonzero(ours != ref)[0]
    assert bad.size == 0, [(float(x[i]), hex(int(ours[i])), hex(int(ref[i]))) for i in bad[:8]]


def test_cast_nan_inf(orc):
    for e, m in [(5, 2), (4, 3), (3, 0), (8, 23), (5, 10)]:
        ci = orc.cast([np.inf, -np.inf, np.nan], e, m)
        d = orc.decode(ci, e, m)
        assert d[0] == np.inf and d[1] == -np.inf
        if m > 0:
            assert np.isnan(d[2])
        else:           # m = 0 has no NaN code; NaN maps to the Inf code (A12)
            assert np.isinf(d[2])


# ---------------------------------------------------------------- brute force

def _all_values(e, m):
    """Every finite non-negative value of (e,m), by code, from the paper's
    definition of the format's range (Table 2) -- built with Fraction-free
    integer arithmetic: value(code) = code-th representable number."""
    bias = (1 << (e - 1)) - 1
    vals = []
    for E in range(0, (1 << e) - 1):
        for M in range(1 << m):
            if E == 0:
                vals.append(math.ldexp(M, 1 - bias - m))
            else:
                vals.append(math.ldexp((1 << m) + M, E - bias - m))
    return np.array(vals, dtype=np.float64), bias


def _brute_force_mag_codes(ax, e, m):
    """argmin_{v in values U {2^(bias+1)}} |v - x| with ties -> even code."""
    vals, bias = _all_values(e, m)
    cand = np.concatenate([vals, [math.ldexp(1.0, bias + 1)]])
    inf_code = ((1 << e) - 1) << m
    out = np.empty(ax.size, dtype=np.uint32)
    for s in range(0, ax.size, 2048):
        a = ax[s:s + 2048, None]
        d = np.abs(cand[None, :] - a)
        dmin = d.min(axis=1, keepdims=True)
        ismin = d == dmin
        # among minima (at most two, adjacent codes), pick the even code
        idx = np.arange(cand.size)[None, :]
        even = ismin & (idx % 2 == 0)
        pick = np.where(even.any(axis=1), np.argmax(even, axis=1), np.argmax(ismin, axis=1))
        code = pick.astype(np.uint32)
        code[pick == vals.size] = inf_code
        code[ax[s:s + 2048] >= math.ldexp(1.0, bias + 1)] = inf_code
        out[s:s + 2048] = code
    return out


SMALL_FORMATS = [(e, m) for e in range(2, 9) for m in range(0, 12 - e)]


@pytest.mark.parametrize("fmt", SMALL_FORMATS, ids=lambda f: f"e{f[0]}m{f[1]}")
def test_cast_brute_force_small_formats(orc, fmt):
    """S:92 / S:410 idea: exhaustive enumeration of every code of tiny formats."""
    e, m = fmt
    vals, bias = _all_values(e, m)
    rng = np.random.default_rng([synthetic.SEED, e, m])
    mids = (vals[1:] + vals[:-1]) / 2
    with np.errstate(over="ignore"):  # probes past fp32 max become inf and are dropped below
        probes = np.concatenate([vals, mids, mids * (1 + 2.0 ** -20), mids * (1 - 2.0 ** -20),
                                 rng.uniform(0, 2.0 ** (bias + 2), 3000),
                                 np.exp2(rng.uniform(-150, min(bias + 2, 127), 3000))]).astype(np.float32)
    probes = np.concatenate([probes, np.nextafter(probes, np.float32(np.inf)),
                             np.nextafter(probes, np.float32(0))])
    probes = probes[np.isfinite(probes)]
    ours = orc.cast(probes, e, m)
    ref = _brute_force_mag_codes(probes.astype(np.float64), e, m)
    bad = np.nonzero(ours != ref)[0]
    assert bad.size == 0, [(float(probes[i]), hex(int(ours[i])), hex(int(ref[i]))) for i in bad[:5]]
    # sign symmetry
    neg = orc.cast(-probes, e, m)
    assert np.array_equal(neg, ours | np.uint32(1 << (e + m)))


def test_cast_brute_force_5_10_sampled(orc):
    e, m = 5, 10
    rng = np.random.default_rng([synthetic.SEED, 510])
    probes = np.exp2(rng.uniform(-26, 17, 6000)).astype(np.float32)
    ours = orc.cast(probes, e, m)
    ref = _brute_force_mag_codes(probes.astype(np.float64), e, m)
    assert np.array_equal(ours, ref)


@pytest.mark.parametrize("fmt", [(3, 0), (5, 2), (4, 3), (5, 6), (5, 10), (8, 7), (2, 1), (6, 9)])
def test_cast_invariants(orc, fmt):
    """idempotence, monotonicity, sign symmetry."""
    e, m = fmt
    x = synthetic.fp32_probe_patterns(200000)
    x = x[np.isfinite(x)]
    c = orc.cast(x, e, m)
    d = orc.decode(c, e, m)
    assert np.array_equal(orc.cast(d, e, m), c)                       # idempotent
    xs = np.sort(x.astype(np.float64)).astype(np.float32)
    ds = orc.decode(orc.cast(xs, e, m), e, m).astype(np.float64)
    assert np.all(ds[1:] >= ds[:-1])                                  # monotone
    assert np.array_equal(orc.cast(-x, e, m), c ^ np.uint32(1 << (e + m)))


def test_hand_roundings_spec_examples(orc):
    """SPEC S:68-71 examples (derived there from a brute-force oracle) and the
    tie cases of readings A9-A11."""
    cast = lambda x, e, m: int(orc.cast([x], e, m)[0])
    assert cast(1.25, 5, 2) == 0x3D
    assert cast(1.125, 5, 2) == 0x3C            # tie 1.0 / 1.25 -> even code (1.0)
    assert cast(65536.0, 5, 2) == 0x7C          # +Inf
    assert cast(2.0 ** -17, 5, 2) == 0x00       # tie 0 / 2^-16 -> 0
    assert cast(1.0, 5, 2) == 0x3C              # S:84 "0b0_01111_00"
    assert cast(57344.0, 5, 2) == 0x7B          # max finite
    assert cast(61440.0, 5, 2) == 0x7C          # overflow tie (A11): odd 0x7B vs even Inf
    assert cast(12.0, 3, 0) == 0x6              # m = 0 overflow tie stays finite (A11)
    assert cast(3.0, 3, 0) == 0x4               # A9: ties to even code
    assert cast(248.0, 4, 3) == 0x78            # (4,3) IEEE-style Inf (A12)
    assert cast(240.0, 4, 3) == 0x77


def test_power_of_two_exactness(orc):
    """Section 3.3.1: scaling by 2^k changes only the exponent, so a
    representable value stays representable and the round trip is exact
    (unscale(scale(0.3, 27), 27) = 0.3)."""
    rng = np.random.default_rng([synthetic.SEED, 33])
    for e, m in [(5, 2), (4, 3), (5, 10), (8, 7)]:
        bias = orc.bias(e)
        codes = rng.integers(0, ((1 << e) - 1) << m, 4000).astype(np.uint32)
        x = orc.decode(codes, e, m)
        x = x[np.abs(x) >= 2.0 ** (1 - bias)]                         # normals
        for k in (-3, -1, 1, 2, 5):
            y = np.ldexp(x.astype(np.float64), k)
            ok = (np.abs(y) >= 2.0 ** (1 - bias)) & (np.abs(y) < 2.0 ** bias)
            yy = y[ok].astype(np.float32)
            assert np.array_equal(orc.decode(orc.cast(yy, e, m), e, m), yy)
    s = orc.scale(0.3, 27)
    assert np.float32(orc.scale(s, -27)) == np.float32(0.3)


def test_scale_matches_ldexpf(orc):
    """O5 / A8: one correctly rounded binary32 result, incl. subnormal results;
    numpy's float32 ldexp is an independent library routine."""
    x = synthetic.fp32_probe_patterns(100000)
    x = x[np.isfinite(x)]
    rng = np.random.default_rng(5)
    ks = rng.integers(-160, 160, x.size)
    with np.errstate(over="ignore"):  # overflow to inf is part of the contract checked
        ref = np.ldexp(x, ks.astype(np.int32))
    ours = np.array([orc.scale(float(a), int(k)) for a, k in zip(x[:20000], ks[:20000])], np.float32)
    r = ref[:20000]
    assert np.array_equal(ours.view(np.uint32), r.view(np.uint32))


# SURVEY 8(c)'s constants table for the config formats, each value re-derived here from the
# format's closed forms (O1: maxfinite = (2 - 2^-m) 2^bias, min normal 2^(1-bias), min
# subnormal 2^(1-bias-m); the overflow threshold is the midpoint between maxfinite and
# 2^(bias+1) and the underflow threshold half the min subnormal, each tie going to the even
# code, A9-A11).  Values are exact in binary64 and in fp32 (all are powers of two or short
# binary fractions within fp32's range).
CONFIG_FORMATS = [(3, 0), (5, 2), (4, 3), (5, 6), (5, 10), (8, 7)]


@pytest.mark.parametrize("fmt", CONFIG_FORMATS, ids=lambda f: f"e{f[0]}m{f[1]}")
def test_survey_constants_table(orc, fmt):
    e, m = fmt
    cast = lambda x: int(orc.cast([x], e, m)[0])
    bias = (1 << (e - 1)) - 1
    maxfinite = (2.0 - 2.0 ** -m) * 2.0 ** bias
    min_normal = 2.0 ** (1 - bias)
    min_sub = 2.0 ** (1 - bias - m)
    max_code = (((1 << e) - 2) << m) | ((1 << m) - 1)
    inf_code = ((1 << e) - 1) << m
    assert orc.bias(e) == bias
    assert float(orc.decode([max_code], e, m)[0]) == maxfinite
    assert float(orc.decode([1 << m], e, m)[0]) == min_normal          # first normal code
    assert float(orc.decode([1], e, m)[0]) == min_sub                    # first subnormal code
    assert cast(maxfinite) == max_code
    # overflow: the midpoint between maxfinite and 2^(bias+1) is a tie; above it is Inf
    mid = (maxfinite + 2.0 ** (bias + 1)) / 2
    tie_to_inf = inf_code % 2 == 0 and max_code % 2 == 1
    assert cast(mid) == (inf_code if tie_to_inf else max_code)
    if mid < 3.4e38:
        assert cast(float(np.nextafter(np.float32(mid), np.float32(np.inf)))) == inf_code
    # underflow: half the min subnormal ties to the even code 0; just above rounds to code 1
    assert cast(min_sub / 2) == 0
    assert cast(float(np.nextafter(np.float32(min_sub / 2), np.float32(np.inf)))) == 1
    assert cast(-min_sub / 2) == 1 << (e + m)                           # -0 code
