// aps_device.cuh -- device helpers shared by the kernels: codecs (generic
// bit-arithmetic, hardware fp8, runtime), 128-bit memory helpers, exact
// power-of-two scaling, packing of 4-code groups and generic-width tiles,
// the exponent of the abs-max (FindMaxExp), f~ and the unscale/average.
#pragma once
#include <cstdint>
#include <climits>

#include "aps_internal.h"
#include "aps_numerics.cuh"

namespace aps {

// ------------------------------------------------------------------ codecs
// Uniform interface: enc(float)->code, dec(code)->float (finite codes),
// dec_any (all codes), b(), and optionally enc4/dec4 for byte codes.
template <int E, int M>
struct CGen {
    static constexpr int kB = 1 + E + M;
    static constexpr bool kVec4 = false;
    __device__ __forceinline__ int b() const { return kB; }
    __device__ __forceinline__ uint32_t enc(float y) const
    {
        constexpr Fmt F = make_fmt(E, M);
        return encode(F, y);
    }
    __device__ __forceinline__ uint32_t enc_q(float y) const  // quantise path (encode_q)
    {
        constexpr Fmt F = make_fmt(E, M);
        return encode_q(F, y);
    }
    __device__ __forceinline__ uint32_t enc_q_dec(float y, float &d) const  // + Cast back
    {
        constexpr Fmt F = make_fmt(E, M);
        return encode_q_dec(F, y, d);
    }
    __device__ __forceinline__ float dec(uint32_t c) const
    {
        constexpr Fmt F = make_fmt(E, M);
        return decode_finite(F, c);
    }
    __device__ __forceinline__ float dec_any(uint32_t c) const
    {
        constexpr Fmt F = make_fmt(E, M);
        return decode(F, c);
    }
};

template <bool E4M3>
struct CHw {
    static constexpr int kB = 8;
    static constexpr bool kVec4 = true;
    __device__ __forceinline__ int b() const { return 8; }
    __device__ __forceinline__ uint32_t enc(float y) const
    {
        return (E4M3 ? cvt_e4m3x2(0.f, y) : cvt_e5m2x2(0.f, y)) & 0xffu;
    }
    __device__ __forceinline__ float dec(uint32_t c) const
    {
        return E4M3 ? e4m3x2_to_f32x2(c & 0xffu).x : e5m2x2_to_f32x2(c & 0xffu).x;
    }
    __device__ __forceinline__ float dec_any(uint32_t c) const { return dec(c); }
    __device__ __forceinline__ uint32_t enc4(float4 v) const
    {
        const uint32_t lo = E4M3 ? cvt_e4m3x2(v.y, v.x) : cvt_e5m2x2(v.y, v.x);
        const uint32_t hi = E4M3 ? cvt_e4m3x2(v.w, v.z) : cvt_e5m2x2(v.w, v.z);
        return lo | (hi << 16);
    }
    __device__ __forceinline__ float4 dec4(uint32_t w) const
    {
        const float2 a = E4M3 ? e4m3x2_to_f32x2(w & 0xffffu) : e5m2x2_to_f32x2(w & 0xffffu);
        const float2 c = E4M3 ? e4m3x2_to_f32x2(w >> 16) : e5m2x2_to_f32x2(w >> 16);
        return make_float4(a.x, a.y, c.x, c.y);
    }
};

// IEEE binary16 = (5,10) and bfloat16 = (8,7) through the hardware converters
// (cvt.rn.f16x2.f32 / cvt.rn.bf16x2.f32: RNE, gradual underflow, IEEE overflow
// -- the same Cast on every non-NaN fp32, reading A12), and binary32 = (8,23),
// where Cast is the identity on every non-NaN fp32.
template <bool BF16>
struct CHw16 {
    static constexpr int kB = 16;
    static constexpr bool kVec4 = true;
    __device__ __forceinline__ int b() const { return 16; }
    __device__ __forceinline__ static uint32_t cvt2(float lo, float hi)
    {
        uint32_t d;
        if constexpr (BF16) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
        else asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
        return d;
    }
    __device__ __forceinline__ static float2 uncvt2(uint32_t w)
    {
        if constexpr (BF16) return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
        __half2 h = *reinterpret_cast<__half2 *>(&w);
        return __half22float2(h);
    }
    __device__ __forceinline__ uint32_t enc(float y) const { return cvt2(y, 0.f) & 0xffffu; }
    __device__ __forceinline__ float dec(uint32_t c) const { return uncvt2(c & 0xffffu).x; }
    __device__ __forceinline__ float dec_any(uint32_t c) const { return dec(c); }
    __device__ __forceinline__ uint2 enc4(float4 v) const { return make_uint2(cvt2(v.x, v.y), cvt2(v.z, v.w)); }
    __device__ __forceinline__ float4 dec4(uint2 w) const
    {
        const float2 a = uncvt2(w.x), c = uncvt2(w.y);
        return make_float4(a.x, a.y, c.x, c.y);
    }
};

struct CF32 {
    static constexpr int kB = 32;
    static constexpr bool kVec4 = false;
    __device__ __forceinline__ int b() const { return 32; }
    __device__ __forceinline__ uint32_t enc(float y) const { return __float_as_uint(y); }
    __device__ __forceinline__ float dec(uint32_t c) const { return __uint_as_float(c); }
    __device__ __forceinline__ float dec_any(uint32_t c) const { return __uint_as_float(c); }
};

struct CRt {
    static constexpr int kB = 0;  // runtime width
    static constexpr bool kVec4 = false;
    Fmt F;
    __device__ __forceinline__ int b() const { return F.b; }
    __device__ __forceinline__ uint32_t enc(float y) const { return encode(F, y); }
    __device__ __forceinline__ uint32_t enc_q(float y) const { return encode_q(F, y); }
    __device__ __forceinline__ uint32_t enc_q_dec(float y, float &d) const { return encode_q_dec(F, y, d); }
    __device__ __forceinline__ float dec(uint32_t c) const { return decode_finite(F, c); }
    __device__ __forceinline__ float dec_any(uint32_t c) const { return decode(F, c); }
};

// ------------------------------------------------------------------ memory helpers
__device__ __forceinline__ float4 ld_stream4(const float4 *p)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// 128-bit loads / stores with L2 cache-policy hints; relaxed / acquire flag loads (gpu scope)
__device__ __forceinline__ float4 ld_keep4(const float4 *p, uint64_t pol)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ float4 ld_hint4(const float4 *p, uint64_t pol)
{
    float4 r;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_hint4(float4 *p, float4 v, uint64_t pol)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_hint(uint32_t *p, uint32_t v, uint64_t pol)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(uint2 *p, uint2 v, uint64_t pol)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_hint(uint4 *p, uint4 v, uint64_t pol)
{
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

// mbarrier (shared memory) helpers: producer / consumer handoff inside a CTA
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
// arrive (release at CTA scope: this thread's prior shared / global writes are visible to a waiter)
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
// non-blocking test of phase `parity` (acquire at CTA scope)
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_addr(b)), "r"(parity) : "memory");
    return ok;
}
// bounded wait (2 s of %globaltimer, then flag bit 2 -> APS_ERR_STATE): a bookkeeping bug must
// never hang the GPU
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity, uint32_t *flag)
{
    uint32_t ok;
    uint64_t t0 = 0;
    for (int it = 0;; ++it) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(smem_addr(b)), "r"(parity) : "memory");
        if (ok) return;
        uint64_t ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        if (it == 0) t0 = ns;
        else if (ns - t0 > 2000000000ull) {
            atomicOr(flag, 2u);
            return;
        }
    }
}

// no second codec (uniform formats)
struct CNone {
    static constexpr int kB = -1;
};
// marker: the control-warp kernel runs the abs-max items only (a1 alone)
struct CAOnly {
    static constexpr int kB = -2;
};

// 4 consecutive fp32 of a layer starting at element e0, zero-filled past n.
__device__ __forceinline__ float4 load_group(const float *g, int64_t e0, int64_t n)
{
    if (e0 + 4 <= n) return ld_stream4(reinterpret_cast<const float4 *>(g + e0));
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e0 + 0 < n) v.x = g[e0 + 0];
    if (e0 + 1 < n) v.y = g[e0 + 1];
    if (e0 + 2 < n) v.z = g[e0 + 2];
    return v;
}

__device__ __forceinline__ void store_group(float *o, int64_t e0, int64_t n, float4 v)
{
    if (e0 + 4 <= n) {
        *reinterpret_cast<float4 *>(o + e0) = v;
        return;
    }
    if (e0 + 0 < n) o[e0 + 0] = v.x;
    if (e0 + 1 < n) o[e0 + 1] = v.y;
    if (e0 + 2 < n) o[e0 + 2] = v.z;
}

// ------------------------------------------------------------------ power-of-two scaling
// y = fl32(x * 2^k) with one rounding (ldexpf semantics, reading A8).  For
// k in [-149, 127] 2^k is an exact fp32 (subnormal below -126) and a single
// FMUL rounds once; outside, the product is formed exactly in fp64 and
// rounded once to fp32.
struct Pow2 {
    float f;
    double d;
    bool wide;
    __device__ __forceinline__ explicit Pow2(int k)
    {
        wide = (k < -149 || k > 127);
        f = (k >= -126) ? __uint_as_float((uint32_t)(k + 127) << 23)
                        : __uint_as_float(1u << ((k + 149) & 31));
        d = __longlong_as_double((long long)(uint64_t)(min(max(k, -1022), 1023) + 1023) << 52);
    }
    __device__ __forceinline__ float apply(float x) const
    {
        return wide ? __double2float_rn((double)x * d) : __fmul_rn(x, f);
    }
    __device__ __forceinline__ float4 apply4(float4 v) const
    {
        return make_float4(apply(v.x), apply(v.y), apply(v.z), apply(v.w));
    }
    // !wide only: one FMUL per element.  Kernels branch on `wide` (uniform per layer) around
    // whole loops -- inside a loop the compiler evaluates both sides of apply() and
    // selects (F2F + DMUL + F2F per element)
    __device__ __forceinline__ float4 apply4_narrow(float4 v) const
    {
        return make_float4(__fmul_rn(v.x, f), __fmul_rn(v.y, f), __fmul_rn(v.z, f), __fmul_rn(v.w, f));
    }
};

// ------------------------------------------------------------------ per-element 4-wide helpers
template <class C>
__device__ __forceinline__ uint32_t enc4_bytes(const C &c, float4 v)
{
    if constexpr (C::kVec4) {
        return c.enc4(v);
    } else {
        return c.enc(v.x) | (c.enc(v.y) << 8) | (c.enc(v.z) << 16) | (c.enc(v.w) << 24);
    }
}

template <class C>
__device__ __forceinline__ float4 dec4_bytes(const C &c, uint32_t w)
{
    if constexpr (C::kVec4) {
        return c.dec4(w);
    } else {
        return make_float4(c.dec(w & 0xffu), c.dec((w >> 8) & 0xffu), c.dec((w >> 16) & 0xffu),
                           c.dec(w >> 24));
    }
}

// packed group of 4 codes for the direct widths
template <int B> struct Word4;
template <> struct Word4<8> { using T = uint32_t; };
template <> struct Word4<16> { using T = uint2; };
template <> struct Word4<32> { using T = uint4; };

template <int B, class C>
__device__ __forceinline__ typename Word4<B>::T pack4(const C &c, float4 v)
{
    if constexpr (B == 8) {
        return enc4_bytes(c, v);
    } else if constexpr (B == 16) {
        if constexpr (C::kB == 16 && C::kVec4) return c.enc4(v);
        else return make_uint2(c.enc(v.x) | (c.enc(v.y) << 16), c.enc(v.z) | (c.enc(v.w) << 16));
    } else {
        return make_uint4(c.enc(v.x), c.enc(v.y), c.enc(v.z), c.enc(v.w));
    }
}

template <int B, class C>
__device__ __forceinline__ float4 unpack4(const C &c, typename Word4<B>::T w)
{
    if constexpr (B == 8) {
        return dec4_bytes(c, w);
    } else if constexpr (B == 16) {
        if constexpr (C::kB == 16 && C::kVec4) return c.dec4(w);
        else return make_float4(c.dec(w.x & 0xffffu), c.dec(w.x >> 16), c.dec(w.y & 0xffffu),
                                c.dec(w.y >> 16));
    } else {
        return make_float4(c.dec(w.x), c.dec(w.y), c.dec(w.z), c.dec(w.w));
    }
}

// ------------------------------------------------------------------ generic-width tile packing
// Tile = 128 codes = 4*b words.  Word w holds bits [32w, 32w+32) of the
// LSB-first code stream.
__device__ __forceinline__ uint32_t assemble_word(const uint32_t *codes, int w, int b)
{
    const int bit0 = w * 32;
    int k = bit0 / b;
    const int off = bit0 - k * b;
    uint64_t acc = (uint64_t)codes[k] >> off;
    int have = b - off;
    ++k;
    while (have < 32 && k < kTile) {
        acc |= (uint64_t)codes[k] << have;
        have += b;
        ++k;
    }
    return (uint32_t)acc;
}

// ------------------------------------------------------------------ generic-width tiles in registers
// For b <= 16 (every C4 width that is not 8/16/32: 4-bit (3,0), 12-bit (5,6), runtime
// formats) a warp packs and unpacks a whole tile in registers.  Lane l owns codes
// 4l..4l+3 = bits [4bl, 4bl + 4b) of the tile's LSB-first stream (<= 64 bits).
//  * unpack: each lane loads the 2-3 words its bits touch straight from memory (lanes
//    sharing a word are served by one request) and funnel-shifts its 4 codes out;
//  * pack: b = 4 and b = 12 pair lanes (16 + 16 bits = one word; 48 + 48 bits = three
//    words) with ONE 32-bit shuffle; other widths assemble word w (held by lane w & 31,
//    register w >> 5) from the lanes its bits come from with 64-bit shuffles.
// No shared memory and no per-tile warp serialisation, so a warp keeps several tiles'
// loads in flight.  B = the compile-time width, or 0 for the runtime b.  Every lane of
// the warp must call the pack functions (shuffles).
constexpr int kRegMaxB = 16;

template <int B>
__device__ __forceinline__ uint64_t lane_bits(uint4 cd, int b_)
{
    const int b = B ? B : b_;
    return (uint64_t)cd.x | ((uint64_t)cd.y << b) | ((uint64_t)cd.z << (2 * b)) | ((uint64_t)cd.w << (3 * b));
}

// word w of the tile whose lanes hold `v` (lane_bits); 0 for w >= 4b
template <int B>
__device__ __forceinline__ uint32_t tile_word(uint64_t v, int b_, int w)
{
    const int b = B ? B : b_, nb = 4 * b;
    const bool wide = nb > 32;
    const int l0 = (32 * w) / nb;            // first lane whose bits reach word w
    const int nl = (32 + nb - 1) / nb + 1;   // lanes one word can touch
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < nl; ++k) {
        const int src = l0 + k;
        uint64_t x = __shfl_sync(0xffffffffu, (uint32_t)v, src & 31);
        if (wide) x |= (uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src & 31) << 32;
        const int off = src * nb - 32 * w;   // position of lane src's bits relative to the word
        if (src < 32 && off < 32) word |= off >= 0 ? (uint32_t)(x << off) : (uint32_t)(x >> -off);
    }
    return word;
}

// the (at most two) words of a tile a lane stores: word i0 = v0, word i1 = v1 (-1: none)
struct TileSlots {
    uint32_t v0, v1;
    int i0, i1;
};

template <int B>
__device__ __forceinline__ TileSlots tile_pack(uint4 cd, int b_, int lane)
{
    const int b = B ? B : b_;
    const uint64_t v = lane_bits<B>(cd, b);
    TileSlots t;
    if constexpr (B == 4) {
        // lanes 2i, 2i+1: 16 + 16 bits = word i (stored by the even lane)
        const uint32_t o = __shfl_xor_sync(0xffffffffu, (uint32_t)v, 1);
        t.v0 = (uint32_t)v | (o << 16);
        t.i0 = (lane & 1) ? -1 : (lane >> 1);
        t.v1 = 0u;
        t.i1 = -1;
    } else if constexpr (B == 12) {
        // lanes 2i, 2i+1: 48 + 48 bits = words 3i, 3i+1, 3i+2 (even lane: 3i and 3i+1,
        // whose high half is the odd lane's low 16 bits; odd lane: 3i+2)
        const uint32_t o = __shfl_xor_sync(0xffffffffu, (uint32_t)v, 1);
        const int i = 3 * (lane >> 1);
        if (lane & 1) {
            t.v0 = (uint32_t)(v >> 16);
            t.i0 = i + 2;
            t.i1 = -1;
            t.v1 = 0u;
        } else {
            t.v0 = (uint32_t)v;
            t.i0 = i;
            t.v1 = (uint32_t)(v >> 32) | (o << 16);
            t.i1 = i + 1;
        }
    } else {
        const int nw = 4 * b;
        t.v0 = tile_word<B>(v, b, lane);
        t.i0 = lane < nw ? lane : -1;
        t.v1 = (nw > 32) ? tile_word<B>(v, b, lane + 32) : 0u;
        t.i1 = (nw > 32 && lane + 32 < nw) ? lane + 32 : -1;
    }
    return t;
}

// store a lane's words with st(word_index, value)
template <class St>
__device__ __forceinline__ void tile_store(const TileSlots &t, St st)
{
    if (t.i0 >= 0) st(t.i0, t.v0);
    if (t.i1 >= 0) st(t.i1, t.v1);
}

// the words a lane's bits touch: w0 = 4bl / 32 and the next one or two
struct TileRaw {
    uint32_t x0, x1, x2;
};

template <int B>
__device__ __forceinline__ constexpr bool tile_needs(int k)
{
    // does some lane's bit range reach word w0 + k?  (runtime widths: assume yes)
    if (B == 0) return true;
    for (int l = 0; l < 32; ++l)
        if ((4 * B * l) % 32 + 4 * B > 32 * k) return true;
    return false;
}

template <int B, class Ld>
__device__ __forceinline__ TileRaw tile_fetch(const uint32_t *tw, int b_, int lane, Ld ld)
{
    const int b = B ? B : b_, nw = 4 * b;
    const int w0 = (lane * 4 * b) >> 5;
    TileRaw r;
    r.x0 = ld(tw + w0);
    r.x1 = (tile_needs<B>(1) && w0 + 1 < nw) ? ld(tw + w0 + 1) : 0u;
    r.x2 = (tile_needs<B>(2) && nw > 32 && w0 + 2 < nw) ? ld(tw + w0 + 2) : 0u;
    return r;
}

// the lane's 4 codes from its words
template <int B>
__device__ __forceinline__ uint4 tile_split(const TileRaw &r, int b_, int lane)
{
    const int b = B ? B : b_, nb = 4 * b;
    const int sh = (lane * nb) & 31;
    const uint32_t lo = __funnelshift_r(r.x0, r.x1, sh);
    const uint32_t hi = nb > 32 ? __funnelshift_r(r.x1, r.x2, sh) : 0u;
    const uint64_t v = lo | ((uint64_t)hi << 32);
    const uint64_t mask = (1ull << b) - 1ull;
    return make_uint4((uint32_t)(v & mask), (uint32_t)((v >> b) & mask), (uint32_t)((v >> (2 * b)) & mask),
                      (uint32_t)((v >> (3 * b)) & mask));
}

struct LdPlain {
    __device__ __forceinline__ uint32_t operator()(const uint32_t *p) const { return *p; }
};

// code k of a tile whose words are in shared memory (words[4b] is a zero pad)
__device__ __forceinline__ uint32_t extract_code(const uint32_t *words, int k, int b)
{
    const int bit = k * b;
    const int w = bit >> 5;
    const int sh = bit & 31;
    const uint32_t v = __funnelshift_r(words[w], words[w + 1], sh);
    return b == 32 ? v : (v & ((1u << b) - 1u));
}

// ------------------------------------------------------------------ a1: absmax + local exponent
__device__ __forceinline__ uint32_t absbits4(float4 v)
{
    const uint32_t a = max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu);
    const uint32_t b = max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu);
    return max(a, b);
}

// E = ceil(log2(N * A)) exactly (N*A is exact in binary64); sentinels for
// an all-zero layer (A3) and non-finite input (A4).  The abs bits of fp32
// are monotone in |x|, so the max is order-independent and bit-exact.
__device__ __forceinline__ int32_t exponent_of(uint32_t abits, int N)
{
    if (abits == 0u) return INT32_MIN;
    if (abits >= 0x7f800000u) return INT32_MAX;
    const double d = (double)__uint_as_float(abits) * (double)N;
    const uint64_t bits = (uint64_t)__double_as_longlong(d);
    const int k = (int)(bits >> 52) - 1023;       // d in [2^k, 2^(k+1))
    return (bits & ((1ull << 52) - 1ull)) ? k + 1 : k;
}

// ------------------------------------------------------------------ a3+a4: scale, cast, pack
__device__ __forceinline__ int scale_exponent(const DevTables &t, int layer, int bias, bool lead)
{
    const int32_t E = t.E_glob[layer];
    int ft = (E == INT32_MIN) ? 0 : bias - E;   // f~ = upper_bound_exp - E (Alg. 1)
    if (E == INT32_MAX) {                        // non-finite somewhere: flag (A4)
        ft = 0;
        if (lead) atomicOr(t.flag, 1u);
    }
    if (lead) t.ftilde[layer] = ft;
    return ft;
}

// ------------------------------------------------------------------ a7: unpack, unscale, average
struct Unscale {
    Pow2 s;
    bool div;       // non-power-of-two N: IEEE division
    float inv_n;    // 2^-log2(N) for power-of-two N
    float n_f;
    bool average;
    bool fast;      // !s.wide && !div: two (or one) FMULs, see apply4_fast
    bool scale_n;   // average by a power-of-two N > 1
    __device__ __forceinline__ Unscale(int ft, int N, int avg) : s(-ft)
    {
        average = avg != 0;
        div = (N & (N - 1)) != 0;
        n_f = (float)N;
        inv_n = div ? 1.f : __uint_as_float((uint32_t)(127 - (31 - __clz(N))) << 23);
        fast = !s.wide && !div;
        scale_n = average && N > 1;
    }
    // fl32(fl32(v 2^-f~) 2^-log2 N): x / N for a power-of-two N is the same correctly
    // rounded result as x * 2^-log2 N (reading A16); valid when `fast`
    __device__ __forceinline__ float apply_fast(float v) const
    {
        const float x = __fmul_rn(v, s.f);
        return scale_n ? __fmul_rn(x, inv_n) : x;
    }
    __device__ __forceinline__ float4 apply4_fast(float4 v) const
    {
        return make_float4(apply_fast(v.x), apply_fast(v.y), apply_fast(v.z), apply_fast(v.w));
    }
    __device__ __forceinline__ float apply(float v) const
    {
        float x = s.apply(v);
        if (average) x = div ? __fdiv_rn(x, n_f) : __fmul_rn(x, inv_n);
        return x;
    }
    __device__ __forceinline__ float4 apply4(float4 v) const
    {
        return make_float4(apply(v.x), apply(v.y), apply(v.z), apply(v.w));
    }
};

// ------------------------------------------------------------------ bounded spin
// Device-side waits (grid barrier, per-layer completion) give up after 2 s of
// %globaltimer and raise flag bit 2 (reported by aps_status_sync as
// APS_ERR_STATE): a bookkeeping bug must never hang the GPU.
constexpr uint32_t kFlagNonfinite = 1u, kFlagWaitTimeout = 2u;
__device__ __forceinline__ uint64_t global_ns()
{
    uint64_t ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    return ns;
}
template <class Ready>
__device__ __forceinline__ void spin_until(Ready ready, uint32_t *flag)
{
    if (ready()) return;
    const uint64_t t0 = global_ns();
    while (!ready()) {
        __nanosleep(32);
        if (global_ns() - t0 > 2000000000ull) {
            atomicOr(flag, kFlagWaitTimeout);
            return;
        }
    }
}

// ------------------------------------------------------------------ dispatch
// Calls f(codec) with the compiled specialisation for the config formats,
// the hardware fp8 codec when requested, else the runtime codec.
template <class F>
cudaError_t with_codec(int e, int m, bool hw, F &&f)
{
    if (hw && e == 5 && m == 2) return f(CHw<false>{});
    if (hw && e == 4 && m == 3) return f(CHw<true>{});
    if (hw && e == 5 && m == 10) return f(CHw16<false>{});
    if (hw && e == 8 && m == 7) return f(CHw16<true>{});
    if (hw && e == 8 && m == 23) return f(CF32{});
    if (e == 5 && m == 2) return f(CGen<5, 2>{});
    if (e == 4 && m == 3) return f(CGen<4, 3>{});
    if (e == 3 && m == 0) return f(CGen<3, 0>{});
    if (e == 5 && m == 6) return f(CGen<5, 6>{});
    if (e == 5 && m == 10) return f(CGen<5, 10>{});
    if (e == 8 && m == 7) return f(CGen<8, 7>{});
    if (e == 8 && m == 23) return f(CGen<8, 23>{});
    CRt c;
    c.F = make_fmt(e, m);
    return f(c);
}

}  // namespace aps
