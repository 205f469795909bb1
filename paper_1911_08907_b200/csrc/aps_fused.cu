// aps_fused.cu -- the whole N = 1 APS sync in ONE launch (SURVEY 8(a) a1 + a3 + a4 + a7):
// FindMaxExp (Alg. 1 line 3), f~ = upper_bound_exp - E (line 4), the scale,
// Cast and pack (lines 5-6), Cast back, unscale and average (lines 8-9,
// P:254-256).  With one rank no collective separates FindMaxExp from Cast, but Cast of
// layer l still needs the abs-max of ALL of layer l.
//
// Schedule: a wavefront over the work items (32 KB of one layer each).  One claim
// counter walks a merged sequence of 2n positions in which the quantise item B(i) trails
// the abs-max item A(i) by D positions, D >= (items of the largest layer) + lag grids:
//   A(0..D-1), then A(D) B(0) A(D+1) B(1) ..., then B(n-D..n-1)
// so every A item a B item needs is claimed earlier, and B re-reads data read only ~D
// items earlier -- from the 126 MB L2 (the DRAM traffic is one read, the codes and the
// output: 8 L + L b / 8 bytes).
//
// Warp specialisation (the round-1 kernel did the claim, descriptor loads, readiness
// check and abs-max fold on thread 0 between the data loads, and all 8 warps waited for
// it at a CTA barrier every item -- measured: the B items alone ran 7 us slower than a
// static grid-stride pass over the same bytes):
//   * 8 DATA warps consume a ring of S slots in shared memory: wait full[s], read the
//     slot's descriptor (addresses, count, f~), load 8 x 128-bit per lane, abs-max (A) or
//     scale + Cast + pack + Cast back + unscale + store (B), arrive on empty[s].  No CTA
//     barrier, no global atomics.
//   * 1 CONTROL warp (lane 0) fills the ring: claims a position (the next claim is issued
//     one slot early), loads the item's descriptor, for a B item waits (acquire, bounded)
//     until every A item of its layer is folded and turns the layer's abs-max into f~,
//     publishes the slot (arrive full[s]); when a slot comes back it folds the slot's
//     A result into amax[layer] (returning atom.max; the count add depends on its value,
//     so it is issued only once the max is performed at L2 -- no fence draining stores)
//     or counts the B item done.
// Counters are SELF-RESETTING: the last B item of a layer clears amax / adone / bdone,
// the CTA holding the launch's final claim clears the claim counter.  A launch needs no
// call index, parity or host-side state, so a captured CUDA graph replays as is.
// Progress: a control warp waiting for a layer keeps folding its own finished slots; a
// B item depends only on A items at earlier positions, each claimed by a CTA that was
// running when it claimed it (no co-residency needed: a plain launch); every wait is
// bounded (2 s -> APS_ERR_STATE).
#include <cstdint>
#include <climits>
#include <algorithm>
#include <type_traits>

#include "aps_device.cuh"

namespace aps {

constexpr int kCwSlots = APS_CW_SLOTS;
// a1 alone: a 4-slot ring, all 4 in flight, data warps take slots two at a time (16
// loads per lane in flight: each warp's 8 x 128-bit loads of one item left ~14 MB in
// flight over the GPU, short of what HBM needs; one slot at a time measured 25.2 us with
// 2 in flight, 26.6 with 3: profiles/r02i_ab_abs.txt)
#ifndef APS_ABS_PAIR
#define APS_ABS_PAIR 0  // 1: 25.7-26.6 us vs 23.4-23.5 (0): profiles/r02n_ab_absmax_pair.txt
#endif
#ifndef APS_ABS_CTAS
#define APS_ABS_CTAS 3
#endif
#ifndef APS_ABS_DEPTH
#define APS_ABS_DEPTH 2
#endif
constexpr int kAbsSlots = APS_ABS_PAIR ? 4 : 3;
constexpr int kAbsDepth = APS_ABS_PAIR ? 4 : APS_ABS_DEPTH;
constexpr int kAbsCtasPerSm = APS_ABS_PAIR ? 2 : APS_ABS_CTAS;  // (two items' loads per lane need the registers)

constexpr int kCwDataWarps = kThreads / 32;            // 8
constexpr int kCwThreads = kThreads + 32;               // + the control warp

struct CwSlot {
    const float *src;
    float *dst;
    int64_t byte_pos;
    int cnt, n_tiles, ft, kind, fmt, layer, litems;  // kind: 0 abs-max (A), 1 quantise (B), 2 end; litems: items of the layer
};

// Generic width b <= 16 (4-bit (3,0), 12-bit (5,6), runtime formats) of a quantise item:
// each data warp owns tiles warp, warp + 8, ... of the item; all its loads are issued
// first (8 x 128-bit per lane in flight, as the byte-code path), then every tile is
// scaled, Cast, packed in registers (warp shuffles, aps_device.cuh) and decoded back.
template <int B, bool FAST, class CC>
__device__ __forceinline__ void cw_quant_reg(const CC &cc, const float *src, float *dst, uint8_t *pk, int cnt,
                                             int n_tiles, bool full, const Pow2 &sc, const Unscale &us,
                                             uint64_t strm, int warp, int lane)
{
    constexpr int kJ = kItemTiles / kCwDataWarps;
    const int b = cc.b();
    uint32_t *outw = reinterpret_cast<uint32_t *>(pk);
    float4 v[kJ];
    if (full) {  // unconditional 128-bit loads: all kJ in flight before the first use
        const float4 *g4 = reinterpret_cast<const float4 *>(src) + lane;
#pragma unroll
        for (int j = 0; j < kJ; ++j) v[j] = ld_hint4(g4 + (warp + j * kCwDataWarps) * (kTile / 4), strm);
    } else {
#pragma unroll
        for (int j = 0; j < kJ; ++j) v[j] = load_group(src, (int64_t)(warp + j * kCwDataWarps) * kTile + lane * 4, cnt);
    }
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
        const int tt = warp + j * kCwDataWarps;
        if (tt >= n_tiles) break;  // warp-uniform
        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
        const float4 y = FAST ? sc.apply4_narrow(v[j]) : sc.apply4(v[j]);
        float4 d;
        const uint4 cd = make_uint4(cc.enc_q_dec(y.x, d.x), cc.enc_q_dec(y.y, d.y), cc.enc_q_dec(y.z, d.z),
                                    cc.enc_q_dec(y.w, d.w));
        uint32_t *tw = outw + (int64_t)tt * (4 * b);
        tile_store(tile_pack<B>(cd, b, lane), [&](int i, uint32_t x) { st_hint(tw + i, x, strm); });
        const float4 o = FAST ? us.apply4_fast(d) : us.apply4(d);
        if (full) st_hint4(reinterpret_cast<float4 *>(dst + e0), o, strm);
        else store_group(dst, e0, cnt, o);
    }
}

template <class C, class C2>
__global__ void __launch_bounds__(kCwThreads, C2::kB == CAOnly::kB ? kAbsCtasPerSm : kCwCtasPerSm)
    fused_cw_kernel(DevTables t, C c, C2 c2, int lag, int bias, int bias2, int fmt2, int avg)
{
    constexpr bool kTwo = C2::kB >= 0;  // items with fmt == fmt2 use c2 (bias2): the hybrid layers
    constexpr bool kAOnly = C2::kB == CAOnly::kB;  // a1 alone (aps_layer_scales): avg carries N
    // items in flight per CTA: a1 alone keeps fewer (its items are short; a deep ring only
    // lengthens the queue every CTA drains at the end of the launch)
    constexpr int kSlots = kAOnly ? kAbsSlots : kCwSlots;
    constexpr int kDepth = kAOnly ? kAbsDepth : kSlots;
    constexpr int NT = kThreads;       // data threads
    constexpr int kPer = kItemTiles * kTile / 4 / NT;  // float4 per data thread per item: 8
    __shared__ CwSlot s_slot[kSlots];
    __shared__ uint32_t s_part[kSlots][kCwDataWarps];     // per-warp abs-max of an A slot
    __shared__ __align__(8) uint64_t s_full[kSlots], s_empty[kSlots];
    __shared__ __align__(16) uint32_t s_codes[kCwDataWarps][kTile];  // generic widths
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n = t.n_items, D = lag, total = kAOnly ? n : 2 * n;
    uint32_t *const amax = t.amax2, *const adone = t.layer_done, *const bdone = t.bdone;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], kCwDataWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kCwDataWarps) {
        // ======================================================== control warp
        if (lane == 0) [&]() {
        auto decode = [&](int j, bool &isB) -> int {
            if (kAOnly || j < D) { isB = false; return j; }
            if (j < total - D) {
                const int k = j - D;
                isB = k & 1;
                return isB ? (k >> 1) : D + (k >> 1);
            }
            isB = true;
            return n - D + (j - (total - D));
        };
        // fold pipeline: the count of the A slot folded last (its add depends on the
        // returned max) and the B item counted last (its returned count decides the reset)
        int pa_layer = -1, pb_layer = -1;
        uint32_t pa_old = 0, pb_old = 0, pb_target = 0;
        auto settle = [&]() {
            if (pa_layer >= 0) {
                const uint32_t inc = (pa_old == 0xffffffffu) ? 0u : 1u;  // always 1: abs bits <= 0x7fffffff
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(&adone[pa_layer]), "r"(inc) : "memory");
                pa_layer = -1;
            }
            if (pb_layer >= 0) {
                if (pb_old == pb_target - 1u) {  // the layer's last B item: reset its counters for the next call
                    amax[pb_layer] = 0u;
                    adone[pb_layer] = 0u;
                    bdone[pb_layer] = 0u;
                }
                pb_layer = -1;
            }
        };
        auto fold = [&](int s) {  // slot s came back from the data warps
            const CwSlot &sl = s_slot[s];
            settle();
            if (sl.kind == 0) {
                uint32_t m = 0;
#pragma unroll
                for (int w = 0; w < kCwDataWarps; ++w) m = max(m, s_part[s][w]);
                if constexpr (kAOnly) {  // no per-layer count: the last CTA finishes (below)
                    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&amax[sl.layer]), "r"(m) : "memory");
                } else {
                    asm volatile("atom.relaxed.gpu.global.max.u32 %0, [%1], %2;" : "=r"(pa_old) : "l"(&amax[sl.layer]), "r"(m)
                                 : "memory");
                    pa_layer = sl.layer;
                }
            } else if (sl.kind == 1) {
                pb_old = atomicAdd(&bdone[sl.layer], 1u);
                pb_target = (uint32_t)sl.litems;
                pb_layer = sl.layer;
            }
        };
        int filled = 0, folded = 0;  // slots published / folded so far (slot i % S)
        auto fold_ready = [&](bool block) {
            while (folded < filled) {
                const int s = folded % kSlots;
                const uint32_t ph = (uint32_t)(folded / kSlots) & 1u;
                if (!block && !mbar_test(&s_empty[s], ph)) break;
                if (block) mbar_wait(&s_empty[s], ph, t.flag);
                fold(s);
                ++folded;
                if (block) break;
            }
        };
        // Claims.  a1 alone: positions 0 .. grid-1 are taken statically (CTA b takes b: no
        // atomic round trip before the first load), later ones are grid + atomicAdd; nothing
        // waits on another CTA there.  The fused kernel claims EVERY position dynamically:
        // a B item waits for the A items of its layer, and a position held by a CTA that is
        // not resident (two APS launches sharing the GPU, each partly resident) could then
        // never be processed.  Either way every CTA makes exactly one claim past the end, so
        // the launch's last claim is total + grid - 1.
        const int64_t claim_off = kAOnly ? (int64_t)gridDim.x : 0;
        int64_t raw = kAOnly ? (int64_t)blockIdx.x : (int64_t)atomicAdd(t.claim64, 1ull);
        for (;;) {
            const int s = filled % kSlots;
            if (filled >= kDepth) {  // at most kDepth items in flight: fold the oldest first
                while (folded <= filled - kDepth) fold_ready(true);
            }
            fold_ready(false);
            const int64_t j = raw;
            if (j >= total) {
                if (j == (int64_t)total + gridDim.x - 1) *t.claim64 = 0ull;  // the launch's final claim
                s_slot[s].kind = 2;
                mbar_arrive(&s_full[s]);
                ++filled;
                break;
            }
            raw = claim_off + (int64_t)atomicAdd(t.claim64, 1ull);  // next claim, in flight while this slot is prepared
            bool isB;
            const int k = decode((int)j, isB);
            const Item it = t.items[k];
            const ItemPtr ip = t.iptr[k];
            CwSlot sl;
            sl.src = ip.src;
            sl.dst = ip.dst;
            sl.byte_pos = it.byte_pos;
            sl.cnt = it.cnt;
            sl.n_tiles = it.n_tiles;
            sl.kind = isB ? 1 : 0;
            sl.fmt = it.fmt;
            sl.layer = it.layer;
            sl.litems = it.layer_items;
            sl.ft = 0;
            if (isB) {
                const uint32_t target = (uint32_t)it.layer_items;
                if (ld_acquire_u32(&adone[it.layer]) < target) {
                    // wait for the layer's A items; keep folding this CTA's own finished slots
                    const uint64_t t0 = global_ns();
                    while (ld_acquire_u32(&adone[it.layer]) < target) {
                        fold_ready(false);
                        settle();
                        __nanosleep(64);
                        if (global_ns() - t0 > 2000000000ull) {
                            atomicOr(t.flag, kFlagWaitTimeout);
                            break;
                        }
                    }
                }
                const int32_t E = exponent_of(ld_relaxed_u32(&amax[it.layer]), 1);
                const int bs = (kTwo && it.fmt == fmt2) ? bias2 : bias;  // the layer's upper_bound_exp
                sl.ft = (E == INT32_MIN || E == INT32_MAX) ? 0 : bs - E;  // f~ (Alg. 1 line 4)
                if (it.tile_begin == 0) {  // record E, f~, the non-finite flag (A4)
                    t.E_local[it.layer] = E;
                    t.ftilde[it.layer] = sl.ft;
                    if (E == INT32_MAX) atomicOr(t.flag, kFlagNonfinite);
                }
            }
            s_slot[s] = sl;
            mbar_arrive(&s_full[s]);
            ++filled;
        }
        while (folded < filled - 1) fold_ready(true);  // (the end slot needs no fold)
        settle();
        }();
        if constexpr (kAOnly) {
            // a1 alone: every A item was folded with a fire-and-forget red.max; the CTA
            // counts itself once (after a fence: cumulativity orders its red.max first),
            // and the last CTA turns the maxima into E_l = ceil(log2(N A_l)) and clears them
            __syncwarp();
            uint32_t last = 0;
            if (lane == 0) {
                __threadfence();
                last = atomicAdd(t.ranges_done, 1u) == gridDim.x - 1u;
                if (last) *t.ranges_done = 0u;
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {
                // the whole GPU waits for this: all loads of a batch in flight at once (a
                // volatile load per layer, each behind the previous store, took ~5 us)
                __threadfence();
                constexpr int kB = 8;
                for (int l0 = 0; l0 < t.n_layers; l0 += 32 * kB) {
                    uint32_t a[kB];
#pragma unroll
                    for (int k = 0; k < kB; ++k) {
                        const int l = l0 + lane + 32 * k;
                        a[k] = l < t.n_layers ? __ldcg(amax + l) : 0u;
                    }
#pragma unroll
                    for (int k = 0; k < kB; ++k) {
                        const int l = l0 + lane + 32 * k;
                        if (l < t.n_layers) {
                            t.E_local[l] = exponent_of(a[k], avg);
                            amax[l] = 0u;
                        }
                    }
                }
            }
        }
        return;
    }

    // ======================================================== data warps
    uint64_t keep, strm;
#ifndef APS_ABS_KEEP_FRAC
#define APS_ABS_KEEP_FRAC 0.5  // a1 alone: fraction of its loads marked evict_last: 0.5 -> quant_pack 16.4 vs 17.2 us (1.0), a1 unchanged (profiles/r02t_ab_keep.txt)
#endif
    if constexpr (kAOnly) {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(keep) : "f"((float)APS_ABS_KEEP_FRAC));
    } else {
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    }
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(strm));
    if constexpr (kAOnly && APS_ABS_PAIR) {
        // a1 alone: two slots at a time (the second may be the end marker)
        auto part_max = [&](const float *src, int cnt) {  // a partial item (a layer's last)
            const float4 *g4 = reinterpret_cast<const float4 *>(src);
            uint32_t mx = 0;
            const int n4 = cnt >> 2;
            for (int q = threadIdx.x; q < n4; q += NT) mx = max(mx, absbits4(ld_hint4(g4 + q, keep)));
            if ((int)threadIdx.x < (cnt & 3)) mx = max(mx, __float_as_uint(src[4 * n4 + threadIdx.x]) & 0x7fffffffu);
            return mx;
        };
        auto finish = [&](int s, uint32_t mx) {
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) s_part[s][warp] = mx;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[s]);
        };
        for (int i = 0;; i += 2) {
            const int s0 = i % kSlots, s1 = (i + 1) % kSlots;
            mbar_wait(&s_full[s0], (uint32_t)(i / kSlots) & 1u, t.flag);
            if (s_slot[s0].kind == 2) break;
            mbar_wait(&s_full[s1], (uint32_t)((i + 1) / kSlots) & 1u, t.flag);
            const bool two = s_slot[s1].kind != 2;
            const float *src0 = s_slot[s0].src, *src1 = s_slot[s1].src;
            const int cnt0 = s_slot[s0].cnt, cnt1 = two ? s_slot[s1].cnt : 0;
            const bool full0 = cnt0 == kItemTiles * kTile, full1 = cnt1 == kItemTiles * kTile;
            float4 v0[kPer], v1[kPer];
            if (full0) {
                const float4 *g4 = reinterpret_cast<const float4 *>(src0) + threadIdx.x;
#pragma unroll
                for (int q = 0; q < kPer; ++q) v0[q] = ld_hint4(g4 + q * NT, keep);
            }
            if (full1) {
                const float4 *g4 = reinterpret_cast<const float4 *>(src1) + threadIdx.x;
#pragma unroll
                for (int q = 0; q < kPer; ++q) v1[q] = ld_hint4(g4 + q * NT, keep);
            }
            uint32_t m0 = 0;
            if (full0) {
#pragma unroll
                for (int q = 0; q < kPer; ++q) m0 = max(m0, absbits4(v0[q]));
            } else {
                m0 = part_max(src0, cnt0);
            }
            finish(s0, m0);
            if (!two) break;
            uint32_t m1 = 0;
            if (full1) {
#pragma unroll
                for (int q = 0; q < kPer; ++q) m1 = max(m1, absbits4(v1[q]));
            } else {
                m1 = part_max(src1, cnt1);
            }
            finish(s1, m1);
        }
        return;
    }
    for (int i = 0;; ++i) {
        const int s = i % kSlots;
        mbar_wait(&s_full[s], (uint32_t)(i / kSlots) & 1u, t.flag);
        const int kind = s_slot[s].kind;
        if (kind == 2) break;
        const float *src = s_slot[s].src;
        const int cnt = s_slot[s].cnt;
        const bool full = cnt == kItemTiles * kTile;
        if (kind == 0) {
            // ---------------- abs-max item
            const float4 *g4 = reinterpret_cast<const float4 *>(src);
            uint32_t mx = 0;
            if (full) {
                float4 v[kPer];
#pragma unroll
                for (int q = 0; q < kPer; ++q) v[q] = ld_hint4(g4 + threadIdx.x + q * NT, keep);
#pragma unroll
                for (int q = 0; q < kPer; ++q) mx = max(mx, absbits4(v[q]));
            } else {
                const int n4 = cnt >> 2;
                for (int q = threadIdx.x; q < n4; q += NT) mx = max(mx, absbits4(ld_hint4(g4 + q, keep)));
                if ((int)threadIdx.x < (cnt & 3)) mx = max(mx, __float_as_uint(src[4 * n4 + threadIdx.x]) & 0x7fffffffu);
            }
            mx = __reduce_max_sync(0xffffffffu, mx);
            if (lane == 0) s_part[s][warp] = mx;
        } else if constexpr (!kAOnly) {
            // ---------------- quantise + unscale item
            float *dst = s_slot[s].dst;
            const int ft = s_slot[s].ft;
            const Pow2 sc(ft);
            const Unscale us(ft, 1, avg);
            uint8_t *pk = t.packed + s_slot[s].byte_pos;
            const int n_tiles = s_slot[s].n_tiles;
            auto quantise = [&](const auto &cc) {
                using CC = std::decay_t<decltype(cc)>;
                constexpr int B = CC::kB;
                if constexpr (B == 8 || B == 16 || B == 32) {
                    using W = typename Word4<B>::T;
                    W *out = reinterpret_cast<W *>(pk);
                    if (full && !sc.wide && us.fast) {
                        const float4 *g4 = reinterpret_cast<const float4 *>(src);
                        float4 *o4 = reinterpret_cast<float4 *>(dst);
                        float4 v[kPer];
#pragma unroll
                        for (int q = 0; q < kPer; ++q) v[q] = ld_hint4(g4 + threadIdx.x + q * NT, strm);
#pragma unroll
                        for (int q = 0; q < kPer; ++q) {
                            const float4 y = make_float4(__fmul_rn(v[q].x, sc.f), __fmul_rn(v[q].y, sc.f),
                                                         __fmul_rn(v[q].z, sc.f), __fmul_rn(v[q].w, sc.f));
                            const W code = pack4<B>(cc, y);
                            st_hint(out + threadIdx.x + q * NT, code, strm);
                            st_hint4(o4 + threadIdx.x + q * NT, us.apply4_fast(unpack4<B>(cc, code)), strm);
                        }
                    } else {
                        const int ng = n_tiles * (kTile / 4);
                        for (int q = threadIdx.x; q < ng; q += NT) {
                            const W code = pack4<B>(cc, sc.apply4(load_group(src, 4 * (int64_t)q, cnt)));
                            out[q] = code;
                            store_group(dst, 4 * (int64_t)q, cnt, us.apply4(unpack4<B>(cc, code)));
                        }
                    }
                } else if constexpr (B > 0) {
                    if (!sc.wide && us.fast) cw_quant_reg<B, true>(cc, src, dst, pk, cnt, n_tiles, full, sc, us, strm, warp, lane);
                    else cw_quant_reg<B, false>(cc, src, dst, pk, cnt, n_tiles, full, sc, us, strm, warp, lane);
                } else if (cc.b() <= kRegMaxB) {
                    if (!sc.wide && us.fast) cw_quant_reg<0, true>(cc, src, dst, pk, cnt, n_tiles, full, sc, us, strm, warp, lane);
                    else cw_quant_reg<0, false>(cc, src, dst, pk, cnt, n_tiles, full, sc, us, strm, warp, lane);
                } else {
                    // runtime widths 17..31: per-warp tile through shared memory
                    const int b = cc.b();
                    uint32_t *codes = s_codes[warp];
                    uint32_t *outw = reinterpret_cast<uint32_t *>(pk);
                    for (int tt = warp; tt < n_tiles; tt += kCwDataWarps) {
                        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
                        const float4 y = sc.apply4(load_group(src, e0, cnt));
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
                if (s_slot[s].fmt == fmt2) quantise(c2);
                else quantise(c);
            } else {
                quantise(c);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[s]);
    }
}

template <class C, class C2>
static int cw_grid(int n_items, int cap)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_cw_kernel<C, C2>, kCwThreads, 0);
    per_sm = std::max(1, std::min(per_sm, kCwCtasPerSm));
    if (cap > 0) per_sm = std::min(per_sm, cap);  // aps_set_occupancy
    return std::max(1, std::min(n_items, sm_count() * per_sm));
}

template <class C, class C2>
static cudaError_t launch_cw(const DevTables &t, C c, C2 c2, int bias, int bias2, int fmt2, int average,
                             int max_layer_items, cudaStream_t s, int cap)
{
    if (t.n_items == 0) return cudaSuccess;
    const int grid = cw_grid<C, C2>(t.n_items, cap);
    int lag = std::min(t.n_items, max_layer_items + kWaveLagGrids * grid);
    // A plain launch: progress needs no co-residency.  A control warp waits only for A
    // items at earlier claim positions, and a position is claimed only by a CTA that is
    // running and publishes it at once into its own slot ring, whose data warps never
    // wait; a waiting control warp keeps folding its finished slots.  CTAs not yet
    // resident hold no claims.  (A cooperative launch would also keep the kernel from
    // sharing SMs with concurrent work -- the DDP hook's backward kernels.)
    fused_cw_kernel<C, C2><<<grid, kCwThreads, 0, s>>>(t, c, c2, lag, bias, bias2, fmt2, average);
    return cudaGetLastError();
}

cudaError_t launch_fused_cw(const DevTables &t, int e, int m, bool hw, int average, int max_layer_items, cudaStream_t s,
                            int ctas_per_sm)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        return launch_cw(t, c, CNone{}, bias, 0, -1, average, max_layer_items, s, ctas_per_sm);
    });
}

// a1 alone (aps_layer_scales, the N > 1 path): the same control-warp schedule over the
// A items only -- dynamic claims (no tail of idle SMs), descriptor and pointer loads off
// the data warps, 3 items per CTA in flight -- and each layer's last A item writes E_l.
cudaError_t launch_absmax_cw(const DevTables &t, int world, cudaStream_t s)
{
    if (t.n_items == 0) return cudaSuccess;
    const int grid = cw_grid<CF32, CAOnly>(t.n_items, kAbsCtasPerSm);
    fused_cw_kernel<CF32, CAOnly><<<grid, kCwThreads, 0, s>>>(t, CF32{}, CAOnly{}, 0, 0, 0, -1, world);
    return cudaGetLastError();
}

cudaError_t launch_fused_cw_hybrid(const DevTables &t, int e, int m, bool hw, int e2, int m2, bool hw2, int fmt2,
                                   int average, int max_layer_items, cudaStream_t s, int ctas_per_sm)
{
    const int bias = (1 << (e - 1)) - 1, bias2 = (1 << (e2 - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        if (e2 == 8 && m2 == 23 && hw2)
            return launch_cw(t, c, CF32{}, bias, bias2, fmt2, average, max_layer_items, s, ctas_per_sm);
        if (e2 == 5 && m2 == 6)  // the paper's 12-bit format: compiled (lane-pair packing), not the runtime codec
            return launch_cw(t, c, CGen<5, 6>{}, bias, bias2, fmt2, average, max_layer_items, s, ctas_per_sm);
        CRt c2;
        c2.F = make_fmt(e2, m2);
        return launch_cw(t, c, c2, bias, bias2, fmt2, average, max_layer_items, s, ctas_per_sm);
    });
}

}  // namespace aps
