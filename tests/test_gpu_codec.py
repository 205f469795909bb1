"""Device codec parity (libaps debug entry points through the C ABI) against
the CPU oracle, element by element, plus exhaustive sweeps over all 2^32 fp32
patterns against torch's dtype conversions where a format equals a torch
dtype.  Needs a B200."""
import numpy as np
import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu

FORMATS = [(5, 2), (4, 3), (3, 0), (5, 6), (5, 10), (8, 7), (8, 23),
           (2, 0), (2, 1), (6, 9), (4, 6), (7, 12), (8, 0), (3, 4), (2, 20), (8, 15)]


@pytest.fixture(scope="module")
def aps():
    import paper_1911_08907_b200 as pkg
    pkg.load()
    torch.cuda.set_device(0)
    return pkg


def _probes(e, m, orc):
    x = synthetic.fp32_probe_patterns(1 << 22)
    b = 1 + e + m
    if b <= 16:   # every midpoint of neighbouring codes and +-1 ulp around it
        vals = orc.decode(np.arange(1 << b, dtype=np.uint32), e, m).astype(np.float64)
        vals = np.unique(vals[np.isfinite(vals)])
        mids = ((vals[1:] + vals[:-1]) / 2).astype(np.float32)
        x = np.concatenate([x, mids, np.nextafter(mids, np.float32(np.inf)),
                            np.nextafter(mids, np.float32(-np.inf)), -mids])
    return x


@pytest.mark.parametrize("fmt", FORMATS, ids=lambda f: f"e{f[0]}m{f[1]}")
def test_debug_cast_vs_oracle(aps, orc, fmt):
    e, m = fmt
    x = _probes(e, m, orc)
    gpu = aps.debug_cast(torch.from_numpy(x).cuda(), e, m).cpu().numpy().view(np.uint32)
    ref = orc.cast(x, e, m)
    bad = np.nonzero(gpu != ref)[0]
    assert bad.size == 0, [(hex(int(x.view(np.uint32)[i])), hex(int(gpu[i])), hex(int(ref[i]))) for i in bad[:8]]


@pytest.mark.parametrize("fmt", [f for f in FORMATS if 1 + f[0] + f[1] <= 16], ids=lambda f: f"e{f[0]}m{f[1]}")
def test_debug_decode_all_codes_vs_oracle(aps, orc, fmt):
    e, m = fmt
    codes = np.arange(1 << (1 + e + m), dtype=np.uint32)
    gpu = aps.debug_decode(torch.from_numpy(codes.view(np.int32)).cuda(), e, m).cpu().numpy()
    ref = orc.decode(codes, e, m)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(gpu), nan)
    assert np.array_equal(gpu[~nan].view(np.uint32), ref[~nan].view(np.uint32))


@pytest.mark.parametrize("fmt,dt", [((5, 2), torch.float8_e5m2), ((5, 10), torch.float16),
                                    ((8, 7), torch.bfloat16)], ids=lambda x: str(x))
def test_debug_cast_exhaustive_vs_torch(aps, fmt, dt):
    """All 2^32 fp32 bit patterns (NaN inputs excluded: payload conventions
    differ) against torch's conversion of the same dtype."""
    e, m = fmt
    chunk = 1 << 28
    for start in range(0, 1 << 32, chunk):
        bits = torch.arange(start, start + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        ours = aps.debug_cast(x, e, m)
        t = x.to(dt)
        ref = (t.view(torch.uint8).to(torch.int32) if t.element_size() == 1
               else t.view(torch.int16).to(torch.int32) & 0xFFFF)
        ok = (ours == ref) | torch.isnan(x)
        assert bool(ok.all()), f"mismatch in chunk {start:#x}"
        del bits, x, ours, t, ref, ok


@pytest.mark.parametrize("fmt", [(5, 2), (4, 3), (5, 10), (8, 7), (8, 23)], ids=lambda f: f"e{f[0]}m{f[1]}")
def test_hw_codec_equals_generic(aps, fmt):
    """The fast codecs equal the generic bit-arithmetic cast.  fp8
    (cvt.rn.satfinite.{e5m2,e4m3}x2): on every fp32 pattern with
    |x| <= 1.5 * 2^bias -- the largest magnitude the APS path can present to a
    cast (scaled values <= 2^bias / N, pre-rounding partial sums <= 2^bias +
    2^bias / N, Eq. (1)), reading A12.  binary16 / bfloat16
    (cvt.rn.{f16,bf16}x2.f32) and binary32 (identity): on EVERY non-NaN fp32
    pattern, +-Inf included.  Exhaustive, both signs; decode on every finite
    code (sampled 2^26 + specials for the 32-bit format)."""
    e, m = fmt
    bias = (1 << (e - 1)) - 1
    b = 1 + e + m
    fp8 = b == 8
    limit = int(np.float32(1.5 * 2.0 ** bias).view(np.uint32)) if fp8 else 0x7F800000
    chunk = 1 << 28
    for start in range(0, limit + 1, chunk):
        stop = min(start + chunk, limit + 1)
        bits = torch.arange(start, stop, dtype=torch.int64, device="cuda").to(torch.int32)
        for sign in (0, -(1 << 31)):
            x = (bits | sign).view(torch.float32)
            a = aps.debug_cast(x, e, m, hw=False)
            c = aps.debug_cast(x, e, m, hw=True)
            assert torch.equal(a, c), f"hw/generic differ in chunk {start:#x} sign {sign}"
            del x, a, c
        del bits
    if b <= 16:
        codes = torch.arange(0, 1 << b, dtype=torch.int32, device="cuda")
    else:
        g = torch.Generator(device="cuda").manual_seed(synthetic.SEED)
        codes = torch.randint(-(1 << 31), (1 << 31) - 1, (1 << 26,), generator=g, device="cuda", dtype=torch.int64)
        special = torch.tensor([0, 1, 0x7FFFFF, 0x800000, 0x7F7FFFFF, 0x3F800000], dtype=torch.int64, device="cuda")
        codes = torch.cat([codes, special, special | (1 << 31)]).to(torch.int32)
    fin = ((codes >> m) & ((1 << e) - 1)) != (1 << e) - 1
    a = aps.debug_decode(codes, e, m, hw=False)
    c = aps.debug_decode(codes, e, m, hw=True)
    assert torch.equal(a[fin].view(torch.int32), c[fin].view(torch.int32))


def _finite_codes(e, m):
    b = 1 + e + m
    c = np.arange(1 << b, dtype=np.uint32)
    return c[((c >> m) & ((1 << e) - 1)) != (1 << e) - 1]


@pytest.mark.parametrize("fmt,hw", [((5, 2), False), ((5, 2), True), ((4, 3), False), ((4, 3), True),
                                    ((3, 0), False), ((2, 1), False), ((5, 6), False), ((5, 10), False),
                                    ((8, 7), False), ((4, 6), False), ((8, 23), False), ((5, 10), True),
                                    ((8, 7), True), ((8, 23), True)],
                         ids=lambda x: str(x))
def test_ring_reduce_vs_oracle(aps, orc, fmt, hw):
    """s <- Cast(fl32(dec(recv) + dec(own))) on packed tiles (a5), against the
    oracle's O8 step, on every pair of finite codes (sampled for b > 8)."""
    e, m = fmt
    b = 1 + e + m
    bias = (1 << (e - 1)) - 1
    fin = _finite_codes(e, m)
    rng = np.random.default_rng([synthetic.SEED, e, m, int(hw)])
    if fin.size <= 256:
        A, B = np.meshgrid(fin, fin)
        A, B = A.ravel(), B.ravel()
    else:
        A = fin[rng.integers(0, fin.size, 1 << 21)]
        B = fin[rng.integers(0, fin.size, 1 << 21)]
    if hw and b == 8:   # fp8 converters: APS regime only (reading A12): |a| + |b| <= 1.5 * 2^bias
        va, vb = orc.decode(A, e, m), orc.decode(B, e, m)
        keep = np.abs(va.astype(np.float64)) + np.abs(vb.astype(np.float64)) <= 1.5 * 2.0 ** bias
        A, B = A[keep], B[keep]
    n = (A.size + 127) // 128 * 128
    A = np.concatenate([A, np.zeros(n - A.size, np.uint32)])
    B = np.concatenate([B, np.zeros(n - B.size, np.uint32)])
    own = torch.from_numpy(orc.pack(A, b)).cuda()
    recv = torch.from_numpy(orc.pack(B, b)).cuda()
    aps.debug_ring_reduce(own, recv, n // 128, e, m, hw=hw)
    got = orc.unpack(own.cpu().numpy(), n, b)
    ref = orc.ring_add_n(B, A, e, m)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, [(hex(int(A[i])), hex(int(B[i])), hex(int(got[i])), hex(int(ref[i]))) for i in bad[:8]]
