// aps_kernels.cu -- the separate-call sm_100a kernels of the APS hot path:
//   (a1  absmax_exp: the control-warp kernel of aps_fused.cu over the abs-max items)
//   a3/a4 quant_pack    f~ = upper_bound_exp - E; Cast(g * 2^f~) ; pack    (Alg. 1)
//   a5  ring_reduce     s <- Cast(fl32(dec(recv) + dec(own)))             (Alg. 1)
//   a7  unpack_unscale  Cast(s, 8, 23) / 2^f~ / N                         (Alg. 1)
// All are HBM-bound streaming kernels (no dense contraction: tensor cores do
// not apply).  Design: one CTA per tile-aligned work item of <= 8192
// elements of one layer (a multi-tensor launch covers every layer), 128-bit
// coalesced loads (ld.global.nc.L1::no_allocate) and coalesced stores;
// b = 8/16/32 pack directly from registers, b <= 16 through register tiles
// (aps_device.cuh), b = 17..31 through a per-warp shared-memory tile.
#include <type_traits>
#include <cstdint>
#include <climits>
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "aps_device.cuh"

namespace aps {

// ------------------------------------------------------------------ a3 + a4: scale, Cast, pack
// One CTA per work item (<= 8192 elements of one layer); items in reverse order: a1
// (forward claims, L2 evict_last loads) read these last, so they are the ones still in L2.
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
    uint32_t *out = reinterpret_cast<uint32_t *>(t.packed + it.byte_pos);
    if (b <= kRegMaxB) {
        // b <= 16: the warp's tiles (warp, warp + 8, ...) loaded first, packed in registers
        constexpr int BB = (C::kB > 0 && C::kB <= kRegMaxB) ? C::kB : 0;
        constexpr int kJ = kItemTiles / (NT / 32);
        float4 v[kJ];
        if (n == kItemTiles * kTile) {  // unconditional 128-bit loads, all in flight before the first use
            const float4 *g4 = reinterpret_cast<const float4 *>(g + begin) + lane;
#pragma unroll
            for (int j = 0; j < kJ; ++j) v[j] = ld_stream4(g4 + (warp + j * (NT / 32)) * (kTile / 4));
        } else {
#pragma unroll
            for (int j = 0; j < kJ; ++j) v[j] = load_group(g + begin, (int64_t)(warp + j * (NT / 32)) * kTile + lane * 4, n);
        }
        auto pass = [&](auto narrow) {  // (branch on s.wide around the loop: see Pow2)
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int tt = warp + j * (NT / 32);
                if (tt >= it.n_tiles) break;  // warp-uniform
                const float4 y = decltype(narrow)::value ? s.apply4_narrow(v[j]) : s.apply4(v[j]);
                const uint4 cd = make_uint4(c.enc_q(y.x), c.enc_q(y.y), c.enc_q(y.z), c.enc_q(y.w));
                uint32_t *tw = out + (int64_t)tt * (4 * b);
                tile_store(tile_pack<BB>(cd, b, lane), [&](int i, uint32_t x) { tw[i] = x; });
            }
        };
        if (!s.wide) pass(std::true_type{});
        else pass(std::false_type{});
        return;
    }
    uint32_t *codes = s_codes[warp];
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
        if (us.fast) {  // (branch around the loop: see Pow2::apply4_narrow)
#pragma unroll
            for (int j = 0; j < kPer; ++j) st_out4(o4 + threadIdx.x + j * NT, us.apply4_fast(unpack4<B>(c, w[j])), pol);
        } else {
#pragma unroll
            for (int j = 0; j < kPer; ++j) st_out4(o4 + threadIdx.x + j * NT, us.apply4(unpack4<B>(c, w[j])), pol);
        }
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
    const uint32_t *in = reinterpret_cast<const uint32_t *>(t.packed + it.byte_pos);
    if (b <= kRegMaxB) {
        // b <= 16: the warp's tiles' words loaded first, split into codes in registers
        constexpr int BB = (C::kB > 0 && C::kB <= kRegMaxB) ? C::kB : 0;
        constexpr int kJ = kItemTiles / (NT / 32);
        TileRaw wr[kJ];
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const int tt = warp + j * (NT / 32);
            wr[j] = tt < it.n_tiles ? tile_fetch<BB>(in + (int64_t)tt * (4 * b), b, lane, LdPlain{}) : TileRaw{0u, 0u, 0u};
        }
        auto pass = [&](auto fast) {
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const int tt = warp + j * (NT / 32);
                if (tt >= it.n_tiles) break;  // warp-uniform
                const uint4 cd = tile_split<BB>(wr[j], b, lane);
                const float4 d = make_float4(c.dec(cd.x), c.dec(cd.y), c.dec(cd.z), c.dec(cd.w));
                const float4 v = decltype(fast)::value ? us.apply4_fast(d) : us.apply4(d);
                const int64_t e0 = (int64_t)tt * kTile + lane * 4;
                if (e0 + 4 <= n) st_out4(reinterpret_cast<float4 *>(o + begin + e0), v, 0);
                else store_group(o + begin, e0, n, v);
            }
        };
        if (us.fast) pass(std::true_type{});
        else pass(std::false_type{});
        return;
    }
    uint32_t *words = s_words[warp];
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
    if (b <= kRegMaxB) {
        constexpr int BB = (C::kB > 0 && C::kB <= kRegMaxB) ? C::kB : 0;
        for (int64_t tt = blockIdx.x * (int64_t)(NT / 32) + warp; tt < n_tiles; tt += warps) {
            uint32_t *ow = o + tt * (4 * b);
            const uint4 ca = tile_split<BB>(tile_fetch<BB>(r + tt * (4 * b), b, lane, LdPlain{}), b, lane);
            const uint4 cb = tile_split<BB>(tile_fetch<BB>(ow, b, lane, LdPlain{}), b, lane);
            const uint4 res = make_uint4(c.enc(__fadd_rn(c.dec(ca.x), c.dec(cb.x))), c.enc(__fadd_rn(c.dec(ca.y), c.dec(cb.y))),
                                         c.enc(__fadd_rn(c.dec(ca.z), c.dec(cb.z))), c.enc(__fadd_rn(c.dec(ca.w), c.dec(cb.w))));
            tile_store(tile_pack<BB>(res, b, lane), [&](int i, uint32_t x) { ow[i] = x; });
        }
        return;
    }
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

// ------------------------------------------------------------------ per-item addresses
// The fused / A-only control warps read each item's gradient and output address from
// one table (rebuilt when the caller's layer pointers change) instead of chaining
// item -> layer -> pointer loads.
__global__ void build_item_ptrs_kernel(DevTables t)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < t.n_items; k += gridDim.x * blockDim.x) {
        const Item it = t.items[k];
        const int64_t begin = (int64_t)it.tile_begin * kTile;
        t.iptr[k] = ItemPtr{t.src[it.layer] + begin, t.dst[it.layer] + begin};
    }
}

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
