// aps_fused.cu -- the whole N = 1 APS sync in ONE launch (SURVEY 8(a) a1 + a3 + a4 + a7):
// FindMaxExp (Alg. 1 line 3), f~ = upper_bound_exp - E (line 4), the scale,
// Cast and pack (lines 5-6), Cast back, unscale and average (lines 8-9,
// P:254-256).  With one rank no collective separates FindMaxExp from Cast, but Cast of
// layer l still needs the abs-max of ALL of layer l.  The kernel is a wavefront over the
// work items (32 KB of one layer each): position p of a static schedule holds the abs-max
// of item p ("A") and the quantise of item p - D ("B"); D >= (items of the largest layer)
// + grid, so every A item a B item needs sits in an earlier iteration of some CTA, and B
// re-reads data read only ~D items (~28 MB) earlier -- from the 126 MB L2.
//
// Work is per WARP (each of the 8 warps of a CTA owns a 4 KB slice of the position's
// items): no CTA barrier, no claim counter.  Per layer, three self-resetting counters:
//   amax[l]   u32 max of |g| bits (atom.max by each A slice)
//   adone[l]  A slices counted (the add depends on the atom.max's returned value, so it
//             is issued only after the max is performed at L2 -- no release fence, which
//             would drain the lane's pending stores)
//   bdone[l]  B slices done; the last one (8 x items of the layer) resets all three,
// so a launch needs no call index or parity: a captured CUDA graph replays as is.
// Progress: a B slice waits (lane 0, acquire, bounded) only on A slices at smaller
// positions; the A part of an iteration precedes its B part, so the smallest waiting
// position always completes (induction); the grid is co-resident (cooperative launch).
#include <cstdint>
#include <climits>
#include <algorithm>
#include <type_traits>

#include "aps_device.cuh"

namespace aps {

template <class C, class C2, int NT>
__global__ void __launch_bounds__(NT, kW2CtasPerSm)
    fused_w2_kernel(DevTables t, C c, C2 c2, int lag, int bias, int bias2, int fmt2, int avg)
{
    constexpr bool kTwo = C2::kB > 0;          // items with fmt == fmt2 use c2 (bias2): hybrid FP32 layer
    constexpr int kW = NT / 32;                // warps = slices per item
    constexpr int kSliceEl = kItemTiles * kTile / kW;  // 1024 elements per slice
    constexpr int kSliceTiles = kItemTiles / kW;       // 8 tiles per slice
    constexpr int kPer = kSliceEl / 4 / 32;            // float4 per lane per slice: 8
    __shared__ __align__(16) uint32_t s_codes[kW][kTile];  // generic widths: one tile of codes per warp
    const int n = t.n_items, D = lag, G = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e_lo = warp * kSliceEl;          // first element of this warp's slice in an item
    uint64_t keep, strm;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(strm));
    uint32_t *const amax = t.amax2, *const adone = t.layer_done, *const bdone = t.bdone;
    // timeline (compile-time flag 16): warp 0's start / end stamps, wait time and waits per CTA
    constexpr bool kTl = (kFusedDefaultFlags & 16) != 0;
    uint64_t tl_t0 = 0, tl_wait = 0, tl_waits = 0, tl_items = 0;
    if (kTl) tl_t0 = global_ns();
    for (int p = blockIdx.x; p < n + D; p += G) {
        // ------------------------------------------------ A: abs-max of slice `warp` of item p
        int a_layer = -1;
        uint32_t a_old = 0;
        if (p < n) {
            const Item it = t.items[p];
            const float4 *g4 = reinterpret_cast<const float4 *>(t.iptr[p].src + e_lo);
            uint32_t mx = 0;
            if (e_lo + kSliceEl <= it.cnt) {
                float4 v[kPer];
#pragma unroll
                for (int q = 0; q < kPer; ++q) v[q] = ld_hint4(g4 + lane + 32 * q, keep);
#pragma unroll
                for (int q = 0; q < kPer; ++q) mx = max(mx, absbits4(v[q]));
            } else if (e_lo < it.cnt) {  // the layer's last, partial slice
                const int cnt = it.cnt - e_lo, n4 = cnt >> 2;
                for (int q = lane; q < n4; q += 32) mx = max(mx, absbits4(ld_hint4(g4 + q, keep)));
                if (lane < (cnt & 3))
                    mx = max(mx, __float_as_uint(t.iptr[p].src[e_lo + 4 * n4 + lane]) & 0x7fffffffu);
            }
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) {
                asm volatile("atom.relaxed.gpu.global.max.u32 %0, [%1], %2;" : "=r"(a_old) : "l"(&amax[it.layer]), "r"(mx)
                             : "memory");
                a_layer = it.layer;
            }
        }
        // ------------------------------------------------ B: quantise + unscale slice `warp` of item p - D
        const int qi = p - D;
        if (qi >= 0) {
            const Item it = t.items[qi];
            const int l = it.layer;
            const bool two = kTwo && it.fmt == fmt2;
            const uint32_t target = (uint32_t)(kW * it.layer_items);
            int ft = 0;
            if (lane == 0) {
                if (kTl && warp == 0 && ld_acquire_u32(&adone[l]) < target) {
                    const uint64_t w0 = global_ns();
                    spin_until([&] { return ld_acquire_u32(&adone[l]) >= target; }, t.flag);
                    tl_wait += global_ns() - w0;
                    ++tl_waits;
                }
                spin_until([&] { return ld_acquire_u32(&adone[l]) >= target; }, t.flag);
                const int32_t E = exponent_of(ld_relaxed_u32(&amax[l]), 1);
                ft = (E == INT32_MIN || E == INT32_MAX) ? 0 : (two ? bias2 : bias) - E;  // f~ (Alg. 1 line 4)
                if (it.tile_begin == 0 && warp == 0) {  // record E, f~, the non-finite flag (A4)
                    t.E_local[l] = E;
                    t.ftilde[l] = ft;
                    if (E == INT32_MAX) atomicOr(t.flag, kFlagNonfinite);
                }
            }
            ft = __shfl_sync(0xffffffffu, ft, 0);
            const Pow2 s(ft);
            const Unscale us(ft, 1, avg);
            const float *src = t.iptr[qi].src + e_lo;
            float *dst = t.iptr[qi].dst + e_lo;
            const int cnt = it.cnt - e_lo;  // valid elements of this slice (may be <= 0)
            auto quantise = [&](const auto &cc) {
                using CC = std::decay_t<decltype(cc)>;
                constexpr int B = CC::kB;
                if constexpr (B == 8 || B == 16 || B == 32) {
                    using W = typename Word4<B>::T;
                    W *out = reinterpret_cast<W *>(t.packed + it.byte_pos) + e_lo / 4;
                    if (cnt >= kSliceEl && !s.wide) {
                        const float4 *g4 = reinterpret_cast<const float4 *>(src);
                        float4 *o4 = reinterpret_cast<float4 *>(dst);
                        float4 v[kPer];
#pragma unroll
                        for (int q = 0; q < kPer; ++q) v[q] = ld_hint4(g4 + lane + 32 * q, strm);
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const float4 y = make_float4(__fmul_rn(v[q].x, s.f), __fmul_rn(v[q].y, s.f),
                                                         __fmul_rn(v[q].z, s.f), __fmul_rn(v[q].w, s.f));
                            const W code = pack4<B>(cc, y);
                            st_hint(out + lane + 32 * q, code, strm);
                            st_hint4(o4 + lane + 32 * q, us.apply4(unpack4<B>(cc, code)), strm);
                        }
                    } else if (cnt > 0) {
                        // the slice's tiles (codes past cnt: +0 padding of the tile)
                        const int ng = min(kSliceTiles, it.n_tiles - warp * kSliceTiles) * (kTile / 4);
                        for (int q = lane; q < ng; q += 32) {
                            const W code = pack4<B>(cc, s.apply4(load_group(src, 4 * (int64_t)q, cnt)));
                            out[q] = code;
                            store_group(dst, 4 * (int64_t)q, cnt, us.apply4(unpack4<B>(cc, code)));
                        }
                    }
                } else if (cnt > 0) {
                    // any width: per-warp tiles of 128 codes through shared memory (16 b bytes each)
                    const int b = cc.b();
                    uint32_t *codes = s_codes[warp];
                    uint32_t *outw = reinterpret_cast<uint32_t *>(t.packed + it.byte_pos) + warp * kSliceTiles * 4 * b;
                    const int nt = min(kSliceTiles, it.n_tiles - warp * kSliceTiles);
                    for (int tt = 0; tt < nt; ++tt) {
                        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
                        const float4 y = s.apply4(load_group(src, e0, cnt));
                        const uint4 cd = make_uint4(cc.enc(y.x), cc.enc(y.y), cc.enc(y.z), cc.enc(y.w));
                        *reinterpret_cast<uint4 *>(codes + lane * 4) = cd;
                        __syncwarp();
                        uint32_t *ow = outw + (int64_t)tt * (4 * b);
                        for (int w2 = lane; w2 < 4 * b; w2 += 32) ow[w2] = assemble_word(codes, w2, b);
                        store_group(dst, e0, cnt,
                                    us.apply4(make_float4(cc.dec(cd.x), cc.dec(cd.y), cc.dec(cd.z), cc.dec(cd.w))));
                        __syncwarp();
                    }
                }
            };
            if constexpr (kTwo) {
                if (two) quantise(c2);
                else quantise(c);
            } else {
                quantise(c);
            }
            if (lane == 0) {  // the last B slice of the layer resets its counters for the next call
                const uint32_t done = atomicAdd(&bdone[l], 1u);
                if (done == target - 1u) {
                    amax[l] = 0u;
                    adone[l] = 0u;
                    bdone[l] = 0u;
                }
            }
        }
        // ------------------------------------------------ count the A slice (its max is at L2 by now)
        if (a_layer >= 0) {
            const uint32_t inc = (a_old == 0xffffffffu) ? 0u : 1u;  // always 1: abs bits <= 0x7fffffff
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&adone[a_layer]), "r"(inc) : "memory");
        }
        if (kTl) ++tl_items;
    }
    if (kTl && threadIdx.x == 0 && blockIdx.x * 4 + 3 < kTimelineSlots) {
        t.timeline[blockIdx.x * 4 + 0] = tl_t0;
        t.timeline[blockIdx.x * 4 + 1] = tl_wait;
        t.timeline[blockIdx.x * 4 + 2] = (tl_waits << 32) | tl_items;
        t.timeline[blockIdx.x * 4 + 3] = global_ns();
    }
}

template <class C, class C2>
static int w2_grid(int n_items)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_w2_kernel<C, C2, kThreads>, kThreads, 0);
    per_sm = std::max(1, std::min(per_sm, kW2CtasPerSm));
    return std::max(1, std::min(n_items, sm_count() * per_sm));
}

template <class C, class C2>
static cudaError_t launch_w2(const DevTables &t, C c, C2 c2, int bias, int bias2, int fmt2, int average, int max_layer_items,
                             cudaStream_t s)
{
    if (t.n_items == 0) return cudaSuccess;
    const int grid = w2_grid<C, C2>(t.n_items);
    int lag = std::min(t.n_items, max_layer_items + kWaveLagGrids * grid);
    void *args[] = {const_cast<DevTables *>(&t), &c, &c2, &lag, &bias, &bias2, &fmt2, &average};
    // co-residency of every CTA is required (static schedule): cooperative launch
    return cudaLaunchCooperativeKernel((const void *)fused_w2_kernel<C, C2, kThreads>, dim3(grid), dim3(kThreads), args,
                                       0, s);
}

cudaError_t launch_fused_w2(const DevTables &t, int e, int m, bool hw, int average, int max_layer_items, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        return launch_w2(t, c, CNone{}, bias, 0, -1, average, max_layer_items, s);
    });
}

cudaError_t launch_fused_w2_hybrid32(const DevTables &t, int e, int m, bool hw, int fmt2, int average,
                                     int max_layer_items, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        return launch_w2(t, c, CF32{}, bias, 127, fmt2, average, max_layer_items, s);
    });
}

}  // namespace aps
