// aps_numerics.cuh -- device-side customised-float codec for sm_100a.
//
// Cast(x, exp_bit, man_bit) of Alg. 1 line 6: round-to-nearest-even
// into an IEEE-style (e,m) float with gradual underflow ("smaller
// than 2^-16 will underflow and cast to 0", reading A10) and IEEE
// overflow ("greater than 2^15 will overflow and cast to INF", A11),
// ties to the even code (A9).  Cast(low_g, 8, 23) of line 8 is `dec`.
//
// Implemented with fp32 bit arithmetic (no tables, no division):
//  * target-normal range:   r = (u + (2^(sh-1) - 1) + lsb) >> sh, re-biased,
//    clamped to the Inf code.  The mantissa carry into the exponent and the
//    overflow-to-Inf both fall out of the integer add.
//  * target-subnormal range: one fp32 add of the magic constant
//    M = 2^(24-bias-m), whose ulp is the format's smallest subnormal, lets the
//    FP adder do the RNE; code = bits(|y| + M) - bits(M).  Needs FTZ off.
//  * decode: shift the code into fp32 position and re-bias; subnormals by
//    one exact fp32 subtraction.
// Hardware fast path (APS regime only, reading A12): (5,2) and (4,3) equal
// the OCP e5m2 / e4m3 encodings below their saturation point, so the
// sm_100a cvt.rn.satfinite.{e5m2,e4m3}x2.f32 and cvt.rn.f16x2.{e5m2,e4m3}x2
// converters are bit-identical there.
//
// This file shares no code with oracle/ (the CPU oracle uses binary64
// bracketing); parity is established by the -m gpu tests.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace aps {

struct Fmt {
    int e, m, b, bias;
    uint32_t sh;           // 23 - m
    uint32_t round_half;   // 2^(sh-1) - 1       (sh >= 1)
    uint32_t rebias;       // (127 - bias) << m
    uint32_t inf_code;     // (2^e - 1) << m
    uint32_t nan_code;     // inf_code | 2^(m-1)  (m >= 1), else inf_code
    uint32_t norm_min;     // fp32 bits of 2^(1-bias): smallest target normal
    uint32_t magic_bits;   // fp32 bits of 2^(24-bias-m)
    uint32_t dec_sub_bits; // fp32 bits of 2^(1-bias) for subnormal decode
    uint32_t sign_shift;   // 31 - (e + m)
    uint32_t mag_mask;     // 2^(e+m) - 1
    uint32_t code_mask;    // 2^b - 1
};

__host__ __device__ constexpr Fmt make_fmt(int e, int m)
{
    Fmt f{};
    f.e = e;
    f.m = m;
    f.b = 1 + e + m;
    f.bias = (1 << (e - 1)) - 1;
    f.sh = 23u - (uint32_t)m;
    f.round_half = f.sh ? ((1u << (f.sh - 1)) - 1u) : 0u;
    f.rebias = (uint32_t)(127 - f.bias) << m;
    f.inf_code = ((1u << e) - 1u) << m;
    f.nan_code = m ? (f.inf_code | (1u << (m - 1))) : f.inf_code;
    f.norm_min = (uint32_t)(128 - f.bias) << 23;
    f.magic_bits = (uint32_t)(127 + 24 - f.bias - m) << 23;
    f.dec_sub_bits = (uint32_t)(128 - f.bias) << 23;
    f.sign_shift = 31u - (uint32_t)(e + m);
    f.mag_mask = (uint32_t)((1ull << (e + m)) - 1ull);
    f.code_mask = (uint32_t)((1ull << f.b) - 1ull);
    return f;
}

// --------------------------------------------------------------- generic
__device__ __forceinline__ uint32_t encode(const Fmt &f, float y)
{
    const uint32_t u = __float_as_uint(y);
    const uint32_t a = u & 0x7fffffffu;
    const uint32_t s = (u >> 31) << (f.e + f.m);
    if (f.m == 23) {                                   // (8,23): identity on finite values
        return (a > 0x7f800000u) ? (s | f.nan_code) : u;
    }
    // target-normal branch
    uint32_t r = (a + f.round_half + ((a >> f.sh) & 1u)) >> f.sh;
    r = min(r - f.rebias, f.inf_code);
    // target-subnormal branch: the FP adder rounds |y| to a multiple of min_sub
    const float t = __fadd_rn(__uint_as_float(a), __uint_as_float(f.magic_bits));
    const uint32_t rs = __float_as_uint(t) - f.magic_bits;
    uint32_t mag = (a >= f.norm_min) ? r : rs;
    mag = (a > 0x7f800000u) ? f.nan_code : mag;
    return s | mag;
}

// Cast on the QUANTISE path only (the scaled gradient y = g 2^f~): |y| <= 2^bias / N by
// Eq. (1)-(4) (A2), so no result overflows, and a non-finite gradient raises the
// deferred flag with unspecified outputs (A4) -- the NaN select and the Inf clamp of
// `encode` are dropped (3 of ~13 integer ops: the generic-width kernels are ALU-bound).
// Identical to `encode` for every finite |y| < 2^(emax + 1).
__device__ __forceinline__ uint32_t encode_q(const Fmt &f, float y)
{
    const uint32_t u = __float_as_uint(y);
    if (f.m == 23) return u;
    const uint32_t a = u & 0x7fffffffu;
    const uint32_t s = (u >> 31) << (f.e + f.m);
    const uint32_t r = ((a + f.round_half + ((a >> f.sh) & 1u)) >> f.sh) - f.rebias;
    const float t = __fadd_rn(__uint_as_float(a), __uint_as_float(f.magic_bits));
    const uint32_t rs = __float_as_uint(t) - f.magic_bits;
    return s | ((a >= f.norm_min) ? r : rs);
}

// encode_q and, from its intermediates, the decoded value (Cast back, Alg. 1 line 8):
// target-normal R0 = (a + half + lsb) >> sh is the rounded value's fp32 bit pattern >> sh,
// so dec = R0 << sh; target-subnormal t = |y| + M is rounded, so dec = t - M exactly.
// Saves re-extracting the fields from the code in the fused kernel (ALU-bound widths).
__device__ __forceinline__ uint32_t encode_q_dec(const Fmt &f, float y, float &dec)
{
    const uint32_t u = __float_as_uint(y);
    if (f.m == 23) {
        dec = y;
        return u;
    }
    const uint32_t a = u & 0x7fffffffu;
    const uint32_t sgn = u & 0x80000000u;
    const uint32_t r0 = (a + f.round_half + ((a >> f.sh) & 1u)) >> f.sh;
    const float t = __fadd_rn(__uint_as_float(a), __uint_as_float(f.magic_bits));
    const bool normal = a >= f.norm_min;
    const uint32_t mag = normal ? r0 - f.rebias : __float_as_uint(t) - f.magic_bits;
    const uint32_t vbits = normal ? (r0 << f.sh) : __float_as_uint(__fsub_rn(t, __uint_as_float(f.magic_bits)));
    dec = __uint_as_float(vbits | sgn);
    return (sgn >> (31 - f.e - f.m)) | mag;
}

__device__ __forceinline__ float decode(const Fmt &f, uint32_t c)
{
    const uint32_t s = ((c >> (f.e + f.m)) & 1u) << 31;
    const uint32_t mag = c & f.mag_mask;
    const uint32_t ef = mag >> f.m;
    const uint32_t shifted = mag << f.sh;
    float v;
    if (ef == 0) {
        v = __fsub_rn(__uint_as_float(shifted + f.dec_sub_bits), __uint_as_float(f.dec_sub_bits));
    } else if (ef == (f.inf_code >> f.m)) {
        v = __uint_as_float(0x7f800000u | ((mag & ((1u << f.m) - 1u)) ? 0x400000u : 0u));
    } else {
        v = __uint_as_float(shifted + ((uint32_t)(127 - f.bias) << 23));
    }
    return __uint_as_float(__float_as_uint(v) | s);
}

// decode when the code is known finite (the APS path never produces Inf/NaN
// codes, Eq. (1) P:347-350 / section 3.3.2): no reserved-exponent branch.
__device__ __forceinline__ float decode_finite(const Fmt &f, uint32_t c)
{
    const uint32_t s = ((c >> (f.e + f.m)) & 1u) << 31;
    const uint32_t mag = c & f.mag_mask;
    const uint32_t shifted = mag << f.sh;
    const float vn = __uint_as_float(shifted + ((uint32_t)(127 - f.bias) << 23));
    const float vs = __fsub_rn(__uint_as_float(shifted + f.dec_sub_bits), __uint_as_float(f.dec_sub_bits));
    const float v = (mag >> f.m) ? vn : vs;
    return __uint_as_float(__float_as_uint(v) | s);
}

// --------------------------------------------------------------- hardware fp8
// cvt.rn.satfinite.e5m2x2.f32 d, a, b : d[15:8] = cvt(a), d[7:0] = cvt(b).
__device__ __forceinline__ uint32_t cvt_e5m2x2(float hi, float lo)
{
    uint16_t d;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(d) : "f"(hi), "f"(lo));
    return d;
}
__device__ __forceinline__ uint32_t cvt_e4m3x2(float hi, float lo)
{
    uint16_t d;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(d) : "f"(hi), "f"(lo));
    return d;
}
__device__ __forceinline__ float2 e5m2x2_to_f32x2(uint32_t two_codes)
{
    uint32_t h2;
    asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)two_codes));
    __half2 h = *reinterpret_cast<__half2 *>(&h2);
    return __half22float2(h);
}
__device__ __forceinline__ float2 e4m3x2_to_f32x2(uint32_t two_codes)
{
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)two_codes));
    __half2 h = *reinterpret_cast<__half2 *>(&h2);
    return __half22float2(h);
}

// --------------------------------------------------------------- codecs
// A codec turns 4 fp32 values into 4 codes and back.  Codec::B is the code
// width; B8 codecs pack 4 codes into one uint32 (byte k = element k).

template <int E, int M>
struct GenericCodec {
    static constexpr int B = 1 + E + M;
    static constexpr Fmt F = make_fmt(E, M);
    __device__ __forceinline__ static uint32_t enc(float y) { return encode(F, y); }
    __device__ __forceinline__ static float dec(uint32_t c) { return decode_finite(F, c); }
    __device__ __forceinline__ static float dec_any(uint32_t c) { return decode(F, c); }
};

template <bool E4M3>
struct HwFp8Codec {
    static constexpr int B = 8;
    static constexpr Fmt F = E4M3 ? make_fmt(4, 3) : make_fmt(5, 2);
    __device__ __forceinline__ static uint32_t enc(float y)
    {
        return (E4M3 ? cvt_e4m3x2(0.f, y) : cvt_e5m2x2(0.f, y)) & 0xffu;
    }
    __device__ __forceinline__ static float dec(uint32_t c)
    {
        return E4M3 ? e4m3x2_to_f32x2(c & 0xffu).x : e5m2x2_to_f32x2(c & 0xffu).x;
    }
    __device__ __forceinline__ static float dec_any(uint32_t c) { return dec(c); }
    __device__ __forceinline__ static uint32_t enc4(float4 v)
    {
        const uint32_t lo = E4M3 ? cvt_e4m3x2(v.y, v.x) : cvt_e5m2x2(v.y, v.x);
        const uint32_t hi = E4M3 ? cvt_e4m3x2(v.w, v.z) : cvt_e5m2x2(v.w, v.z);
        return lo | (hi << 16);
    }
    __device__ __forceinline__ static float4 dec4(uint32_t w)
    {
        const float2 a = E4M3 ? e4m3x2_to_f32x2(w & 0xffffu) : e5m2x2_to_f32x2(w & 0xffffu);
        const float2 b = E4M3 ? e4m3x2_to_f32x2(w >> 16) : e5m2x2_to_f32x2(w >> 16);
        return make_float4(a.x, a.y, b.x, b.y);
    }
};

// Runtime (e,m) codec for formats without a compiled specialisation.
struct RuntimeCodec {
    Fmt F;
    __device__ __forceinline__ uint32_t enc(float y) const { return encode(F, y); }
    __device__ __forceinline__ float dec(uint32_t c) const { return decode_finite(F, c); }
    __device__ __forceinline__ float dec_any(uint32_t c) const { return decode(F, c); }
};

}  // namespace aps
