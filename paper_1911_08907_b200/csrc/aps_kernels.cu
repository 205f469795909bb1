// aps_kernels.cu -- the sm_100a kernels of the APS hot path:
//   a1  absmax_exp      FindMaxExp(g * N) for every layer, one launch      (Alg. 1)
//   a3/a4 quant_pack    f~ = upper_bound_exp - E; Cast(g * 2^f~) ; pack    (Alg. 1)
//   a5  ring_reduce     s <- Cast(fl32(dec(recv) + dec(own)))             (Alg. 1)
//   a7  unpack_unscale  Cast(s, 8, 23) / 2^f~ / N                         (Alg. 1)
// All are HBM-bound streaming kernels (no dense contraction: tensor cores do
// not apply).  Design: one CTA per tile-aligned work item of <= 8192
// elements of one layer (a multi-tensor launch covers every layer), 128-bit
// coalesced loads (ld.global.nc.L1::no_allocate) and coalesced stores;
// b = 8/16/32 pack directly from registers, other widths go through a
// per-warp shared-memory tile.
#include <type_traits>
#include <cstdint>
#include <climits>
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "aps_device.cuh"

namespace aps {

// ------------------------------------------------------------------ a1: abs-max, balanced stream
// FindMaxExp (Alg. 1 line 3; function P:260-271) for every layer in ONE launch of
// exactly kAbsCtasPerSm x SMs CTAs.  The layers are laid end to end in "vector space"
// (vector = 4 consecutive fp32 of one layer; layer l owns vectors [voff[l], voff[l+1]),
// its last vector partial when numel % 4 != 0) and CTA b streams the equal share
// [b V / G, (b+1) V / G): every SM moves the same number of bytes, so the launch has no
// tail of idle SMs (the round-1 kernel, one CTA per 4 work items, left SMs idle 23 % of
// its time: profiles/r02a_absmax_raw.csv).  A share is walked in chunks of 8 x NT
// vectors (8 independent 128-bit loads in flight per thread):
//   * chunk inside one layer (the common case): a running per-thread max of that layer,
//     folded into amax[layer] (warp max, one red.max per warp) when the layer changes;
//   * chunk crossing layer boundaries or holding a partial vector: each vector finds its
//     layer (binary search over voff) and is folded with a shared-memory atomicMax into
//     a per-chunk table, flushed with red.max.
// The max of u32 abs bits is order-independent, so the result is bit-exact whatever the
// split.  Completion: one fence by thread 0 after the CTA barrier, one count; the last
// CTA turns the maxima into E_l = ceil(log2(N A_l)) and clears them (self-resetting:
// capture-safe).  Gradients are loaded with an L2 evict_last hint so that quant_pack's
// re-read (reverse order) hits L2.
constexpr int kAbsChunk = 8 * kThreads;  // vectors per chunk (32 KB)

template <int NT>
__global__ void __launch_bounds__(NT, kAbsCtasPerSm) absmax_stream_kernel(DevTables t, int N)
{
    constexpr int kChunk = 8 * NT;
    __shared__ uint32_t s_tab[kChunk];  // slow path: max per layer of the chunk (index layer - l0)
    __shared__ int s_last;
    const int lane = threadIdx.x & 31;
    uint64_t keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    const int64_t V = t.voff[t.n_layers];
    const int64_t lo = V * (int64_t)blockIdx.x / gridDim.x, hi = V * (int64_t)(blockIdx.x + 1) / gridDim.x;
    int l = t.cta_layer[blockIdx.x];  // layer holding vector lo
    for (int k = threadIdx.x; k < kChunk; k += NT) s_tab[k] = 0u;
    __syncthreads();
    uint32_t run = 0;                 // this thread's running max of layer `l` (fast path)
    for (int64_t c0 = lo; c0 < hi; c0 += kChunk) {
        const int64_t c1 = min(hi, c0 + kChunk);
        while (t.voff[l + 1] <= c0) {   // advance to the layer holding c0 (flush the old one)
            const uint32_t m = __reduce_max_sync(0xffffffffu, run);
            if (lane == 0 && m)
                asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&t.amax[l]), "r"(m) : "memory");
            run = 0;
            ++l;
        }
        const int64_t base = t.voff[l];
        const int64_t full_end = base + (t.layers[l].numel >> 2);  // first partial vector (or voff[l+1])
        if (c1 <= full_end) {
            // ---- fast path: the chunk lies in layer l's full vectors
            const float4 *g4 = reinterpret_cast<const float4 *>(t.src[l]);
            const int64_t i0 = c0 - base, i1 = c1 - base;  // vector indices within the layer
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t i = i0 + threadIdx.x + q * NT;
                v[q] = i < i1 ? ld_keep4(g4 + i, keep) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) run = max(run, absbits4(v[q]));
            continue;
        }
        // ---- slow path: layers l .. lh meet the chunk (lh < l + kChunk)
        {
            const uint32_t m = __reduce_max_sync(0xffffffffu, run);
            if (lane == 0 && m)
                asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&t.amax[l]), "r"(m) : "memory");
            run = 0;
        }
        int lh = l;
        {   // last layer meeting the chunk: largest layer with voff <= c1 - 1
            int a = l, b = min(t.n_layers - 1, l + kChunk - 1);
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (t.voff[mid] <= c1 - 1) a = mid; else b = mid - 1;
            }
            lh = a;
        }
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
            const int64_t i = c0 + threadIdx.x + q * NT;
            if (i >= c1) break;
            int a = l, b = lh;   // layer of vector i
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (t.voff[mid] <= i) a = mid; else b = mid - 1;
            }
            const int64_t e0 = 4 * (i - t.voff[a]);         // first element of the vector in layer a
            const int64_t n = t.layers[a].numel;
            const float *g = t.src[a];
            uint32_t mx;
            if (e0 + 4 <= n) {
                mx = absbits4(ld_keep4(reinterpret_cast<const float4 *>(g + e0), keep));
            } else {
                mx = 0;
                for (int64_t e = e0; e < n; ++e) mx = max(mx, __float_as_uint(g[e]) & 0x7fffffffu);
            }
            if (mx) atomicMax(&s_tab[a - l], mx);
        }
        __syncthreads();
        for (int k = threadIdx.x; k <= lh - l; k += NT) {
            const uint32_t m = s_tab[k];
            if (m) {
                asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&t.amax[l + k]), "r"(m) : "memory");
                s_tab[k] = 0u;
            }
        }
        __syncthreads();
        l = lh;  // (the next chunk starts at or after layer lh)
    }
    {
        const uint32_t m = __reduce_max_sync(0xffffffffu, run);
        if (lane == 0 && m && l < t.n_layers)
            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&t.amax[l]), "r"(m) : "memory");
    }
    // completion: the CTA barrier orders every warp's red.max before thread 0's fence
    // (cumulativity), whose count the last CTA acquires
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(t.ranges_done, 1u) == gridDim.x - 1u;
        if (s_last) *t.ranges_done = 0u;  // every CTA of this launch has counted itself
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int k = threadIdx.x; k < t.n_layers; k += NT) {
            uint32_t a_;
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(a_) : "l"(&t.amax[k]) : "memory");
            t.E_local[k] = exponent_of(a_, N);
            t.amax[k] = 0u;
        }
    }
}

template <int B, class C, int NT>
__global__ void __launch_bounds__(NT) quant_pack_direct_kernel(DevTables t, C c, int bias)
{
    const Item it = t.items[t.n_items - 1 - blockIdx.x];  // reverse: a1 read these last (L2)
    const LayerDev L = t.layers[it.layer];
    const float *g = t.src[it.layer];
    const int ft = scale_exponent(t, it.layer, bias, it.tile_begin == 0 && threadIdx.x == 0);
    const Pow2 s(ft);
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    const int64_t n = min((int64_t)it.n_tiles * kTile, L.numel - begin);
    using W = typename Word4<B>::T;
    W *out = reinterpret_cast<W *>(t.packed + it.byte_pos);
    const float *gb = g + begin;
    constexpr int kFull4 = kItemTiles * kTile / 4;
    constexpr int kPer = kFull4 / NT;
    if (n == kItemTiles * kTile && !s.wide) {
        float4 v[kPer];
        const float4 *g4 = reinterpret_cast<const float4 *>(gb);
#pragma unroll
        for (int j = 0; j < kPer; ++j) v[j] = ld_stream4(g4 + threadIdx.x + j * NT);
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const float4 y = make_float4(__fmul_rn(v[j].x, s.f), __fmul_rn(v[j].y, s.f),
                                         __fmul_rn(v[j].z, s.f), __fmul_rn(v[j].w, s.f));
            out[threadIdx.x + j * NT] = pack4<B>(c, y);
        }
    } else {
        const int ng = it.n_tiles * (kTile / 4);
        for (int gi = threadIdx.x; gi < ng; gi += NT) {
            const float4 v = load_group(gb, (int64_t)gi * 4, n);
            out[gi] = pack4<B>(c, s.apply4(v));
        }
    }
}

// any width: per-warp tile through shared memory
template <class C, int NT>
__global__ void __launch_bounds__(NT) quant_pack_tile_kernel(DevTables t, C c, int bias)
{
    __shared__ __align__(16) uint32_t s_codes[NT / 32][kTile];
    const Item it = t.items[t.n_items - 1 - blockIdx.x];  // reverse: a1 read these last (L2)
    const LayerDev L = t.layers[it.layer];
    const float *g = t.src[it.layer];
    const int ft = scale_exponent(t, it.layer, bias, it.tile_begin == 0 && threadIdx.x == 0);
    const Pow2 s(ft);
    const int b = c.b();
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    const int64_t n = min((int64_t)it.n_tiles * kTile, L.numel - begin);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *codes = s_codes[warp];
    uint32_t *out = reinterpret_cast<uint32_t *>(t.packed + it.byte_pos);
    for (int tt = warp; tt < it.n_tiles; tt += NT / 32) {
        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
        const float4 y = s.apply4(load_group(g + begin, e0, n));
        *reinterpret_cast<uint4 *>(codes + lane * 4) =
            make_uint4(c.enc(y.x), c.enc(y.y), c.enc(y.z), c.enc(y.w));
        __syncwarp();
        uint32_t *ow = out + (int64_t)tt * (4 * b);
        for (int w = lane; w < 4 * b; w += 32) ow[w] = assemble_word(codes, w, b);
        __syncwarp();
    }
}

#ifndef APS_UNPACK_HINT
#define APS_UNPACK_HINT 2  // measured: plain 23.5 us, evict_first 21.1 us, .cs 21.0 us (profiles/r01_ab_unpack_store_hint.txt)
#endif
// output store of the unpack pass: 0 plain, 1 L2 evict_first policy, 2 .cs (streaming)
__device__ __forceinline__ void st_out4(float4 *p, float4 v, uint64_t pol)
{
    if constexpr (APS_UNPACK_HINT == 1) {
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
                     "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                     : "memory");
    } else if constexpr (APS_UNPACK_HINT == 2) {
        asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
    } else {
        (void)pol;
        *p = v;
    }
}

template <int B, class C, int NT>
__global__ void __launch_bounds__(NT) unpack_unscale_direct_kernel(DevTables t, C c, int N, int avg)
{
    uint64_t pol = 0;
    if constexpr (APS_UNPACK_HINT == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const Item it = t.items[blockIdx.x];
    const LayerDev L = t.layers[it.layer];
    float *o = t.dst[it.layer];
    const Unscale us(t.ftilde[it.layer], N, avg);
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    const int64_t n = min((int64_t)it.n_tiles * kTile, L.numel - begin);
    using W = typename Word4<B>::T;
    const W *in = reinterpret_cast<const W *>(t.packed + it.byte_pos);
    float *ob = o + begin;
    constexpr int kFull4 = kItemTiles * kTile / 4;
    constexpr int kPer = kFull4 / NT;
    if (n == kItemTiles * kTile) {
        W w[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) w[j] = in[threadIdx.x + j * NT];
        float4 *o4 = reinterpret_cast<float4 *>(ob);
#pragma unroll
        for (int j = 0; j < kPer; ++j) st_out4(o4 + threadIdx.x + j * NT, us.apply4(unpack4<B>(c, w[j])), pol);
    } else {
        const int64_t ng = (n + 3) / 4;
        for (int64_t gi = threadIdx.x; gi < ng; gi += NT)
            store_group(ob, gi * 4, n, us.apply4(unpack4<B>(c, in[gi])));
    }
}

template <class C, int NT>
__global__ void __launch_bounds__(NT) unpack_unscale_tile_kernel(DevTables t, C c, int N, int avg)
{
    __shared__ __align__(16) uint32_t s_words[NT / 32][kTile + 1];
    const Item it = t.items[blockIdx.x];
    const LayerDev L = t.layers[it.layer];
    float *o = t.dst[it.layer];
    const Unscale us(t.ftilde[it.layer], N, avg);
    const int b = c.b();
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    const int64_t n = min((int64_t)it.n_tiles * kTile, L.numel - begin);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *words = s_words[warp];
    const uint32_t *in = reinterpret_cast<const uint32_t *>(t.packed + it.byte_pos);
    for (int tt = warp; tt < it.n_tiles; tt += NT / 32) {
        const uint32_t *iw = in + (int64_t)tt * (4 * b);
        for (int w = lane; w < 4 * b; w += 32) words[w] = iw[w];
        if (lane == 0) words[4 * b] = 0u;
        __syncwarp();
        const int k0 = lane * 4;
        const float4 v = make_float4(c.dec(extract_code(words, k0, b)), c.dec(extract_code(words, k0 + 1, b)),
                                     c.dec(extract_code(words, k0 + 2, b)), c.dec(extract_code(words, k0 + 3, b)));
        store_group(o + begin, (int64_t)tt * kTile + k0, n, us.apply4(v));
        __syncwarp();
    }
}

// ------------------------------------------------------------------ a5: ring reduce step
// own[i] <- Cast(fl32(dec(recv[i]) + dec(own[i])))   (re-quantise after the add, A13)
template <int B, class C, int NT>
__global__ void __launch_bounds__(NT) ring_reduce_direct_kernel(uint8_t *own, const uint8_t *recv,
                                                                 int64_t n_vec, C c)
{
    // one 16-byte vector of codes per thread and iteration (16 codes at b = 8)
    using W = typename Word4<B>::T;
    constexpr int G = 16 / sizeof(W);  // 4-code groups per vector
    uint4 *o = reinterpret_cast<uint4 *>(own);
    const uint4 *r = reinterpret_cast<const uint4 *>(recv);
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n_vec; i += (int64_t)gridDim.x * NT) {
        uint4 va = r[i], vb = o[i];
        W wa[G], wb[G];
        memcpy(wa, &va, 16);
        memcpy(wb, &vb, 16);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float4 a = unpack4<B>(c, wa[g]);
            const float4 b = unpack4<B>(c, wb[g]);
            wb[g] = pack4<B>(c, make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                                            __fadd_rn(a.w, b.w)));
        }
        memcpy(&vb, wb, 16);
        o[i] = vb;
    }
}

template <class C, int NT>
__global__ void __launch_bounds__(NT) ring_reduce_tile_kernel(uint8_t *own, const uint8_t *recv,
                                                               int64_t n_tiles, C c)
{
    __shared__ __align__(16) uint32_t s_a[NT / 32][kTile + 1];
    __shared__ __align__(16) uint32_t s_b[NT / 32][kTile + 1];
    const int b = c.b();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *wa = s_a[warp], *wb = s_b[warp];
    uint32_t *o = reinterpret_cast<uint32_t *>(own);
    const uint32_t *r = reinterpret_cast<const uint32_t *>(recv);
    const int64_t warps = (int64_t)gridDim.x * (NT / 32);
    for (int64_t tt = blockIdx.x * (int64_t)(NT / 32) + warp; tt < n_tiles; tt += warps) {
        uint32_t *ow = o + tt * (4 * b);
        const uint32_t *rw = r + tt * (4 * b);
        for (int w = lane; w < 4 * b; w += 32) {
            wa[w] = rw[w];
            wb[w] = ow[w];
        }
        if (lane == 0) wa[4 * b] = wb[4 * b] = 0u;
        __syncwarp();
        uint32_t res[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = lane * 4 + j;
            res[j] = c.enc(__fadd_rn(c.dec(extract_code(wa, k, b)), c.dec(extract_code(wb, k, b))));
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) wa[lane * 4 + j] = res[j];  // reuse as code array
        __syncwarp();
        for (int w = lane; w < 4 * b; w += 32) ow[w] = assemble_word(wa, w, b);
        __syncwarp();
    }
}

// ------------------------------------------------------------------ fused p = 1 (LDG engine)
// One rank: no collective separates FindMaxExp from Cast, so ONE persistent
// cooperative launch (kFusedCtasPerSm CTAs per SM) does
//   phase A  abs-max of every work item (forward order, L2 evict_last hint):
//            each warp folds its max into the layer with red.max;
//   barrier  each CTA fences once and bumps the done counter; all CTAs wait
//            for the call's target (acquire);
//   phase B  per item in REVERSE order (the most recently read data is still
//            in the 126 MB L2): E_l from the accumulator, f~, scale, Cast,
//            pack (codes -> packed buffer), Cast back, unscale -> output.
// Accumulators are double-buffered by call parity: buffer g&1 is used,
// buffer (g+1)&1 is cleared by the layer's first item for the next call.
__global__ void build_item_ptrs_kernel(DevTables t)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < t.n_items; k += gridDim.x * blockDim.x) {
        const Item it = t.items[k];
        const int64_t begin = (int64_t)it.tile_begin * kTile;
        t.iptr[k] = ItemPtr{t.src[it.layer] + begin, t.dst[it.layer] + begin};
    }
}

#ifndef APS_DIAG_NOWAIT
#define APS_DIAG_NOWAIT 0
#endif
#ifndef APS_DIAG_NOA
#define APS_DIAG_NOA 0
#endif
// ------------------------------------------------------------------ sim: MAX exchange of E
struct PtrArr {
    const int32_t *src[64];
    int32_t *dst[64];
};

__global__ void sim_max_kernel(PtrArr a, int p, int n_layers)
{
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n_layers; l += gridDim.x * blockDim.x) {
        int32_t m = INT32_MIN;
        for (int r = 0; r < p; ++r) m = max(m, a.src[r][l]);
        for (int r = 0; r < p; ++r) a.dst[r][l] = m;
    }
}

// ------------------------------------------------------------------ debug
template <class C>
__global__ void debug_cast_kernel(const float *in, uint32_t *codes, int64_t n, C c)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        codes[i] = c.enc(in[i]);
}

template <class C>
__global__ void debug_decode_kernel(const uint32_t *codes, float *out, int64_t n, C c)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = c.dec_any(codes[i]);
}

int sm_count()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int absmax_grid() { return std::min(kAbsMaxCtas, sm_count() * kAbsCtasPerSm); }

cudaError_t launch_absmax(const DevTables &t, int world, cudaStream_t s)
{
    if (t.n_items == 0) return cudaSuccess;
    absmax_stream_kernel<kThreads><<<absmax_grid(), kThreads, 0, s>>>(t, world);
    return cudaGetLastError();
}

cudaError_t launch_quant_pack(const DevTables &t, int e, int m, bool hw, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        const int b = 1 + e + m;
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32) {
            quant_pack_direct_kernel<C::kB, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
        } else if constexpr (C::kB == 0) {
            if (b == 8) quant_pack_direct_kernel<8, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
            else if (b == 16) quant_pack_direct_kernel<16, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
            else if (b == 32) quant_pack_direct_kernel<32, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
            else quant_pack_tile_kernel<C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
        } else {
            quant_pack_tile_kernel<C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, bias);
        }
        return cudaGetLastError();
    });
}

cudaError_t launch_unpack_unscale(const DevTables &t, int e, int m, bool hw, int world, int average,
                                  cudaStream_t s)
{
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        const int b = 1 + e + m;
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32) {
            unpack_unscale_direct_kernel<C::kB, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
        } else if constexpr (C::kB == 0) {
            if (b == 8) unpack_unscale_direct_kernel<8, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
            else if (b == 16) unpack_unscale_direct_kernel<16, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
            else if (b == 32) unpack_unscale_direct_kernel<32, C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
            else unpack_unscale_tile_kernel<C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
        } else {
            unpack_unscale_tile_kernel<C, kThreads><<<t.n_items, kThreads, 0, s>>>(t, c, world, average);
        }
        return cudaGetLastError();
    });
}

cudaError_t launch_ring_reduce(uint8_t *own, const uint8_t *recv, int64_t n_tiles, int e, int m,
                               bool hw, cudaStream_t s)
{
    if (n_tiles <= 0) return cudaSuccess;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        const int b = 1 + e + m;
        const int64_t n_vec = n_tiles * 16 * b / 16;  // 16-byte vectors (a tile is 16 b bytes)
        const int grid_direct = (int)std::min<int64_t>((n_vec + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
        const int grid_tile = (int)std::min<int64_t>((n_tiles + kThreads / 32 - 1) / (kThreads / 32), (int64_t)sm_count() * 8);
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32) {
            ring_reduce_direct_kernel<C::kB, C, kThreads><<<grid_direct, kThreads, 0, s>>>(own, recv, n_vec, c);
        } else if constexpr (C::kB == 0) {
            if (b == 8) ring_reduce_direct_kernel<8, C, kThreads><<<grid_direct, kThreads, 0, s>>>(own, recv, n_vec, c);
            else if (b == 16) ring_reduce_direct_kernel<16, C, kThreads><<<grid_direct, kThreads, 0, s>>>(own, recv, n_vec, c);
            else if (b == 32) ring_reduce_direct_kernel<32, C, kThreads><<<grid_direct, kThreads, 0, s>>>(own, recv, n_vec, c);
            else ring_reduce_tile_kernel<C, kThreads><<<grid_tile, kThreads, 0, s>>>(own, recv, n_tiles, c);
        } else {
            ring_reduce_tile_kernel<C, kThreads><<<grid_tile, kThreads, 0, s>>>(own, recv, n_tiles, c);
        }
        return cudaGetLastError();
    });
}

// ------------------------------------------------------------------ fused p = 1, wavefront schedule
// No grid barrier: ONE claim counter walks a merged sequence of 2n items in
// which quantise item B(i) trails abs-max item A(i) by `lag` positions:
//   A(0..D-1), then A(D) B(0) A(D+1) B(1) ..., then B(n-D..n-1).
// Every warp of an A item counts itself into the layer's completion counter
// with a fire-and-forget red.release (after its red.max); B(i) waits
// (acquire) until its layer's counter reaches 8 x layer_items for this call.
// With D >= (items of the largest layer) + grid, every A item of B(i)'s layer
// sits earlier in the sequence and is normally finished when B(i) is
// claimed, and B(i) re-reads data read only ~D items (~D x 32 KB) ago: it is
// still in L2.  Progress: a waiting B depends only on A items at earlier
// positions, and each CTA holds at most its current and next claim, so the
// earliest waiting B always completes (induction on position).
// No second codec (uniform formats, or one launch per format group).

// GRAPH = false: per-call state (claim base, call index, accumulator parity) comes from
// the host as launch arguments (the fastest form).  GRAPH = true (capture-safe): the
// call index is derived on the device from a 64-bit claim counter that advances by
// exactly adv = 2 n + kWaveOvershoot * grid per call, so a captured CUDA graph replays
// exactly; measured ~1 us slower per call (profiles/r01_ab_wave_graph_safe.txt).
template <class C, class C2, bool GRAPH, int NT>
__global__ void __launch_bounds__(NT, kWaveCtasPerSm)
    fused_p1_wave_kernel(DevTables t, C c, C2 c2, uint32_t *amax_h, uint32_t *amax_next_h, uint32_t claim_base,
                         uint32_t call_no_h, unsigned long long adv, int lag, int bias, int bias2, int fmt2, int avg,
                         int flags)
{
    // (graph mode keeps its call state in shared memory, not registers: the kernel sits at
    // its 64-register budget)
    __shared__ uint32_t s_call;
    __shared__ unsigned long long s_base64;  // claim counter value at this call's start
    if (GRAPH && threadIdx.x == 0) s_base64 = ~0ull;
    auto amax_of = [&](uint32_t next) -> uint32_t * {
        if constexpr (GRAPH) return t.amax2 + (size_t)((s_call + next) & 1u) * t.n_layers;
        else return next ? amax_next_h : amax_h;
    };
    auto call_no = [&]() -> uint32_t {
        if constexpr (GRAPH) return s_call;
        else return call_no_h;
    };
    constexpr bool kTwo = C2::kB > 0;  // items with fmt == fmt2 use c2 (bias2)
    __shared__ __align__(16) uint32_t s_codes[NT / 32][kTile];
    __shared__ int s_claim[3], s_ft[3], s_ok[3];  // claims run two items ahead (3 slots)
    __shared__ Item s_item[3];                    // ... with their descriptors and addresses, loaded by
    __shared__ ItemPtr s_iptr[3];                 //     thread 0 at claim time (no dependent load at item start)
    __shared__ uint32_t s_part[2][NT / 32];       // per-warp maxima of the last two items
    __shared__ int s_part_layer[2];               // their layer (-1: a quantise item)
    // positions: A(0..D-1), A(D) B(0) A(D+1) B(1) ..., B(n-D..n-1)
    const int n = t.n_items, D = lag, total = 2 * n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool f_st_hint = flags & 64;
    const bool f_timeline = (flags & 16) && blockIdx.x * 4 + 3 < kTimelineSlots;
    auto stamp = [&](int k) {
        if (f_timeline && threadIdx.x == 0) {
            uint64_t ns;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
            t.timeline[blockIdx.x * 4 + k] = ns;
        }
    };
    stamp(0);
    uint64_t tl_wait_ns = 0, tl_waits = 0, tl_items = 0;  // timeline (flag 16): B-item waits of thread 0
    uint64_t keep, strm;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(strm));
    constexpr int kPer = kItemTiles * kTile / 4 / NT;
    constexpr int kFlushThread = 32;  // lane 0 of warp 1 folds finished abs-max items into the layer
    auto decode = [&](int j, bool &isB) -> int {
        if (j < D) { isB = false; return j; }
        if (j < total - D) {
            const int k = j - D;
            isB = k & 1;
            return isB ? (k >> 1) : D + (k >> 1);
        }
        isB = true;
        return n - D + (j - (total - D));
    };
    auto ft_of = [&](const Item &it) -> int {
        const int32_t E = exponent_of(ld_relaxed_u32(&amax_of(0)[it.layer]), 1);
        const int bs = (kTwo && it.fmt == fmt2) ? bias2 : bias;  // the layer's upper_bound_exp
        return (E == INT32_MIN || E == INT32_MAX) ? 0 : bs - E;  // f~ (Alg. 1 line 4)
    };
    auto layer_target = [&](const Item &it) -> uint32_t { return (call_no() + 1u) * (uint32_t)(8 * it.layer_items); };
    // thread 0: claim a position into slot sl; resolve f~ now if it is a quantise item of a complete layer
    auto claim_into = [&](int sl) {
        int j;
        if constexpr (GRAPH) {
            const unsigned long long raw = atomicAdd(t.claim64, 1ull);  // the wavefront's own counter
            if (s_base64 == ~0ull) {  // first claim of this CTA: the call index (one division per CTA)
                const unsigned long long cn = raw / adv;
                s_base64 = cn * adv;
                s_call = (uint32_t)cn;
            }
            j = (int)(raw - s_base64);
        } else {
            j = (int)(atomicAdd(&t.claim[2], 1u) - claim_base);
        }
        s_claim[sl] = j;
        s_ok[sl] = APS_DIAG_NOWAIT;  // (diagnostic build: never wait, results invalid)
        if (APS_DIAG_NOWAIT) s_ft[sl] = 0;
        if (j < total) {
            bool isB;
            const int k = decode(j, isB);
            const Item it = t.items[k];
            s_item[sl] = it;
            s_iptr[sl] = t.iptr[k];
            if (isB) {
                if ((int)(ld_acquire_u32(&t.layer_done[it.layer]) - layer_target(it)) >= 0) {
                    s_ft[sl] = ft_of(it);
                    s_ok[sl] = 1;
                }
            }
        }
    };
    // flush pipeline (kFlushThread): an item's max is folded in (returning atomic) one
    // iteration after the item, and counted (add dependent on the atomic's result, so
    // only after the max is performed at L2) one iteration after that
    int pend_layer = -1;  // layer whose max was folded last iteration and is not yet counted
    uint32_t pend_old = 0;
    auto flush = [&](int pp) {
        if (pend_layer >= 0) {
            const uint32_t inc = (pend_old == 0xffffffffu) ? 0u : 8u;  // always 8: abs bits <= 0x7fffffff
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&t.layer_done[pend_layer]), "r"(inc)
                         : "memory");
            pend_layer = -1;
        }
        const int l = pp >= 0 ? s_part_layer[pp] : -1;
        if (l >= 0) {
            uint32_t m = 0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) m = max(m, s_part[pp][w]);
            asm volatile("atom.relaxed.gpu.global.max.u32 %0, [%1], %2;"
                         : "=r"(pend_old) : "l"(&amax_of(0)[l]), "r"(m) : "memory");
            pend_layer = l;
        }
    };
    if (threadIdx.x == 0) {
        claim_into(0);
        claim_into(1);
        s_part_layer[0] = s_part_layer[1] = -1;
    }
    __syncthreads();
    int slot = 0, par = 0;
    for (int j = s_claim[0]; j < total;) {
        bool isB;
        decode(j, isB);
        const Item it = s_item[slot];
        const ItemPtr p = s_iptr[slot];
        const float4 *g4 = reinterpret_cast<const float4 *>(p.src);
        const bool full = it.cnt == kItemTiles * kTile;
        float4 v[kPer];
        if (full) {
#pragma unroll
            for (int q = 0; q < kPer; ++q) v[q] = ld_hint4(g4 + threadIdx.x + q * NT, isB ? strm : keep);
        }
        if (threadIdx.x == 0) claim_into((slot + 2) % 3);
        if (threadIdx.x == kFlushThread) flush(par ^ 1);
        if (!isB && APS_DIAG_NOA) {
            if (threadIdx.x == 0) s_part_layer[par] = -1;  // (diagnostic build: abs-max items skipped)
        } else if (!isB) {
            // ---------------- abs-max item
            uint32_t mx = 0;
            if (full) {
#pragma unroll
                for (int q = 0; q < kPer; ++q) mx = max(mx, absbits4(v[q]));
            } else {
                const int n4 = it.cnt >> 2;
                for (int q = threadIdx.x; q < n4; q += NT) mx = max(mx, absbits4(ld_hint4(g4 + q, keep)));
                if ((int)threadIdx.x < (it.cnt & 3)) mx = max(mx, __float_as_uint(p.src[4 * n4 + threadIdx.x]) & 0x7fffffffu);
            }
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) s_part[par][warp] = mx;
            if (threadIdx.x == 0) s_part_layer[par] = it.layer;
        } else {
            if (threadIdx.x == 0) s_part_layer[par] = -1;
            // ---------------- quantise + unscale item
            if (!s_ok[slot]) {  // (uniform) layer not seen complete at claim time: wait now
                // this CTA's own not-yet-counted abs-max item may be one the wait needs:
                // count it first (deadlock otherwise)
                if (threadIdx.x == kFlushThread) flush(-1);
                if (threadIdx.x == 0) {
                    const uint64_t w0 = f_timeline ? global_ns() : 0;
                    spin_until([&] { return (int)(ld_acquire_u32(&t.layer_done[it.layer]) - layer_target(it)) >= 0; },
                               t.flag);
                    s_ft[slot] = ft_of(it);
                    if (f_timeline) {
                        tl_wait_ns += global_ns() - w0;
                        ++tl_waits;
                    }
                }
                __syncthreads();
            }
            const int ft = s_ft[slot];
            if (it.tile_begin == 0 && threadIdx.x == 0) {  // record E, f~, flag; clear the next call's accumulator
                const int32_t E = exponent_of(ld_relaxed_u32(&amax_of(0)[it.layer]), 1);
                t.E_local[it.layer] = E;
                t.ftilde[it.layer] = ft;
                if (E == INT32_MAX) atomicOr(t.flag, 1u);
                amax_of(1)[it.layer] = 0u;
            }
            const Pow2 s(ft);
            const Unscale us(ft, 1, avg);
            auto quantise = [&](const auto &cc) {
                using CC = std::decay_t<decltype(cc)>;
                constexpr int B = CC::kB;
                if constexpr (B == 8 || B == 16 || B == 32) {
                    using W = typename Word4<B>::T;
                    W *out = reinterpret_cast<W *>(t.packed + it.byte_pos);
                    if (full && !s.wide) {
                        float4 *o4 = reinterpret_cast<float4 *>(p.dst);
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const float4 y = make_float4(__fmul_rn(v[q].x, s.f), __fmul_rn(v[q].y, s.f),
                                                         __fmul_rn(v[q].z, s.f), __fmul_rn(v[q].w, s.f));
                            const W code = pack4<B>(cc, y);
                            const float4 r = us.apply4(unpack4<B>(cc, code));
                            if (f_st_hint) {
                                st_hint(out + threadIdx.x + q * NT, code, strm);
                                st_hint4(o4 + threadIdx.x + q * NT, r, strm);
                            } else {
                                out[threadIdx.x + q * NT] = code;
                                o4[threadIdx.x + q * NT] = r;
                            }
                        }
                    } else {
                        const int ng = it.n_tiles * (kTile / 4);
                        for (int q = threadIdx.x; q < ng; q += NT) {
                            const W code = pack4<B>(cc, s.apply4(load_group(p.src, 4 * (int64_t)q, it.cnt)));
                            out[q] = code;
                            store_group(p.dst, 4 * (int64_t)q, it.cnt, us.apply4(unpack4<B>(cc, code)));
                        }
                    }
                } else {
                    const int b = cc.b();
                    uint32_t *codes = s_codes[warp];
                    uint32_t *outw = reinterpret_cast<uint32_t *>(t.packed + it.byte_pos);
                    for (int tt = warp; tt < it.n_tiles; tt += NT / 32) {
                        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
                        const float4 y = s.apply4(load_group(p.src, e0, it.cnt));
                        const uint4 cd = make_uint4(cc.enc(y.x), cc.enc(y.y), cc.enc(y.z), cc.enc(y.w));
                        *reinterpret_cast<uint4 *>(codes + lane * 4) = cd;
                        __syncwarp();
                        uint32_t *ow = outw + (int64_t)tt * (4 * b);
                        for (int w2 = lane; w2 < 4 * b; w2 += 32) ow[w2] = assemble_word(codes, w2, b);
                        store_group(p.dst, e0, it.cnt,
                                    us.apply4(make_float4(cc.dec(cd.x), cc.dec(cd.y), cc.dec(cd.z), cc.dec(cd.w))));
                        __syncwarp();
                    }
                }
            };
            if constexpr (kTwo) {
                if (it.fmt == fmt2) quantise(c2);
                else quantise(c);
            } else {
                quantise(c);
            }
        }
        __syncthreads();
        slot = (slot + 1) % 3;
        par ^= 1;
        j = s_claim[slot];
        if (f_timeline) ++tl_items;
    }
    if (threadIdx.x == kFlushThread) {  // drain: the last item's max, then its count
        flush(par ^ 1);
        flush(-1);
    }
    if (f_timeline && threadIdx.x == 0) {
        t.timeline[blockIdx.x * 4 + 1] = tl_wait_ns;
        t.timeline[blockIdx.x * 4 + 2] = (tl_waits << 32) | tl_items;
    }
    stamp(3);
}

template <class C, class C2>
static cudaError_t launch_wave(const DevTables &t, C c, C2 c2, int bias, int bias2, int fmt2, int average,
                               const WaveCall &w, int lag, int grid, cudaStream_t s, bool cooperative)
{
    auto kern = w.graph ? fused_p1_wave_kernel<C, C2, true, kThreads> : fused_p1_wave_kernel<C, C2, false, kThreads>;
    int flags = kFusedDefaultFlags;  // compile time (-DAPS_FUSED_FLAGS=...: timeline stamps, A/B builds)
    unsigned long long adv = 2ull * (unsigned long long)t.n_items + (unsigned long long)kWaveOvershoot * grid;
    uint32_t *cur = t.amax2 + (size_t)(w.gen & 1u) * t.n_layers;
    uint32_t *other = t.amax2 + (size_t)((w.gen + 1u) & 1u) * t.n_layers;
    uint32_t claim_base = w.claim_base, call_no = w.call_no;
    void *args[] = {const_cast<DevTables *>(&t), &c, &c2, &cur, &other, &claim_base, &call_no, &adv, &lag, &bias,
                    &bias2, &fmt2, &average, &flags};
    // co-residency is not needed for progress (a CTA waits only on positions claimed
    // earlier, i.e. by running CTAs); a plain launch lets a concurrent group's kernel
    // fill this one's tail
    if (!cooperative) return cudaLaunchKernel((const void *)kern, dim3(grid), dim3(kThreads), args, 0, s);
    return cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_fused_p1_wave(const DevTables &t, int e, int m, bool hw, int average, const WaveCall &w, int lag,
                                 int grid, cudaStream_t s, bool cooperative)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        return launch_wave(t, c, CNone{}, bias, 0, -1, average, w, lag, grid, s, cooperative);
    });
}

cudaError_t launch_fused_p1_wave_hybrid32(const DevTables &t, int e, int m, bool hw, int fmt2, int average,
                                          const WaveCall &w, int lag, int grid, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        return launch_wave(t, c, CF32{}, bias, 127, fmt2, average, w, lag, grid, s, true);
    });
}

int fused_p1_wave_grid(int e, int m, bool hw, int n_items)
{
    int per_sm = 0;
    with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_p1_wave_kernel<C, CNone, false, kThreads>,
                                                             kThreads, 0);
    });
    per_sm = std::max(1, std::min(per_sm, kWaveCtasPerSm));
    return std::max(1, std::min(n_items, sm_count() * per_sm));
}

cudaError_t launch_build_item_ptrs(const DevTables &t, cudaStream_t s)
{
    build_item_ptrs_kernel<<<(t.n_items + 255) / 256, 256, 0, s>>>(t);
    return cudaGetLastError();
}

cudaError_t launch_sim_max(int32_t *const *E_glob, const int32_t *const *E_local, int p, int n_layers,
                           cudaStream_t s)
{
    if (p > 64) return cudaErrorInvalidValue;
    PtrArr a{};
    for (int r = 0; r < p; ++r) {
        a.src[r] = E_local[r];
        a.dst[r] = E_glob[r];
    }
    sim_max_kernel<<<(n_layers + 255) / 256, 256, 0, s>>>(a, p, n_layers);
    return cudaGetLastError();
}

cudaError_t launch_debug_cast(const float *in, uint32_t *codes, int64_t n, int e, int m, bool hw,
                              cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
        debug_cast_kernel<<<grid, 256, 0, s>>>(in, codes, n, c);
        return cudaGetLastError();
    });
}

cudaError_t launch_debug_decode(const uint32_t *codes, float *out, int64_t n, int e, int m, bool hw,
                                cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
        debug_decode_kernel<<<grid, 256, 0, s>>>(codes, out, n, c);
        return cudaGetLastError();
    });
}

}  // namespace aps
