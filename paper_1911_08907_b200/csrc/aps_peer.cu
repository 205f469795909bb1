// aps_peer.cu -- the all-reduce of Alg. 1 line 7 over PEER MEMORY
// (NVLink / NVSwitch load-store through CUDA IPC mappings) instead of NCCL
// send/recv, with any reduction order and accumulator:
//
//   * owner-computes: rank r reduces ring chunk r (tiles [r T'/p, (r+1) T'/p))
//     by loading the p ranks' packed codes of the chunk directly (p-1 of them
//     over NVLink), folding them in the order the reduction schedule fixes,
//     and STORING the reduced codes into every rank's packed buffer (the
//     all-gather, fused into the same pass).  NVLink bytes per rank equal the
//     ring's: (p-1)/p of the packed buffer in, (p-1)/p out.  No partial sum
//     ever travels, so the order of the additions is a free parameter:
//       - flat ring (reading A14): chunk c accumulated over ranks c+1, ..., c;
//       - hierarchical (reading A23): groups of k consecutive
//         ranks; group chunk c1 = t / (T'/k) accumulated over members
//         c1+1, ..., c1; master chunk c2 = t / (T'/G) over groups c2+1, ..., c2;
//     and the accumulator may be wider than the wire format, or Kahan-
//     compensated (CPD, reading A24) at no wire cost.
//   * cross-rank synchronisation by monotone epoch flags in each rank's
//     workspace, written remotely with st.release.sys after a system fence
//     and polled locally with ld.acquire.sys; every wait is bounded (2 s
//     watchdog -> flag bit 2 -> APS_ERR_STATE), so a missing peer cannot hang
//     the GPU.
//   * AllReduce(max_grad_exp, MAX) (Alg. 1 line 4) the same way: every
//     rank stores its E vector into every rank's slot [rank] (double-buffered
//     by epoch parity), flags, and each rank takes the max of the p slots.
//
// The same kernels serve p simulated ranks on one device (the "peer" pointers
// are then the other contexts' workspaces): the parity tests drive them there.
#include <cstdint>
#include <climits>
#include <algorithm>
#include <cstring>

#include "aps_device.cuh"
#include "aps_peer.h"

namespace aps {

// ------------------------------------------------------------------ system-scope flag helpers
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Peer loads: weak, L1-bypassing.  The codes were published before this kernel
// started (the preceding wait kernel acquired every rank's ready flag at system
// scope, and stream order carries that into this kernel); nothing else writes
// them while this kernel runs (only the owner of a chunk reads or writes it).
__device__ __forceinline__ uint4 ld_peer16(const void *p)
{
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_peer4(const void *p)
{
    uint32_t r;
    asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
// end of a reduce CTA: its remote stores are made visible system-wide once
// (bar.sync orders the CTA's stores before thread 0's fence; the signal kernel
// that follows fences again before it raises the done flag)
// APS_PEER_FENCE: 0 = fence.sc.sys (__threadfence_system), 1 = fence.acq_rel.sys (a release
// fence is all the pattern needs: prior stores before the later flag store) -- A/B
#ifndef APS_PEER_FENCE
#define APS_PEER_FENCE 1
#endif
__device__ __forceinline__ void fence_release_sys()
{
    if constexpr (APS_PEER_FENCE == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else __threadfence_system();
}
__device__ __forceinline__ void cta_fence_system()
{
    __syncthreads();
    if (threadIdx.x == 0) fence_release_sys();
}

__device__ __forceinline__ int32_t ld_relaxed_i32(const int32_t *p)
{
    int32_t v;
    asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// wait until flags[slot + q] >= epoch for every rank q (bounded)
__device__ void wait_all(const PeerArgs &a, int slot, uint32_t epoch, uint32_t *err_flag)
{
    const uint32_t *f = a.flags[a.rank] + slot;
    for (int q = 0; q < a.p; ++q) {
        // a peer may lag by far more than a kernel's own bookkeeping (stragglers, a rank
        // still starting up): this bound is the transport's, not the 2 s kernel watchdog
        if ((int32_t)(ld_acquire_sys(f + q) - epoch) >= 0) continue;
        const uint64_t t0 = global_ns();
        while ((int32_t)(ld_acquire_sys(f + q) - epoch) < 0) {
            __nanosleep(64);
            if (global_ns() - t0 > a.timeout_ns) {
                atomicOr(err_flag, kFlagWaitTimeout);
                return;
            }
        }
    }
}

// ------------------------------------------------------------------ AllReduce(E, MAX)
// post: the next E epoch; E_local -> slot [epoch & 1][rank] of every rank, then flag kSlotE.
__global__ void peer_post_E_kernel(PeerArgs a, const int32_t *E_local, int n_layers)
{
    __shared__ uint32_t s_epoch;
    uint32_t *mine = a.flags[a.rank];
    if (threadIdx.x == 0) s_epoch = mine[kMineE] + 1u;
    __syncthreads();
    const uint32_t epoch = s_epoch;
    const size_t par = (size_t)(epoch & 1u) * (size_t)a.p + (size_t)a.rank;
    for (int q = 0; q < a.p; ++q) {
        int32_t *dst = a.eslots[q] + par * (size_t)n_layers;
        for (int l = threadIdx.x; l < n_layers; l += blockDim.x) dst[l] = E_local[l];
    }
    __syncthreads();  // the CTA's stores precede thread 0's fence and releases (cumulativity)
    if (threadIdx.x == 0) {
        mine[kMineE] = epoch;
        __threadfence_system();
        for (int q = 0; q < a.p; ++q) st_release_sys(a.flags[q] + kSlotE + a.rank, epoch);
    }
}

// collect: wait for every rank's post of this rank's current E epoch, E_glob = max over the slots.
__global__ void peer_collect_E_kernel(PeerArgs a, int32_t *E_glob, int n_layers, uint32_t *err_flag)
{
    const uint32_t epoch = a.flags[a.rank][kMineE];
    if (threadIdx.x == 0) wait_all(a, kSlotE, epoch, err_flag);
    __syncthreads();
    const int32_t *base = a.eslots[a.rank] + (size_t)(epoch & 1u) * (size_t)a.p * (size_t)n_layers;
    for (int l = threadIdx.x; l < n_layers; l += blockDim.x) {
        int32_t mx = INT32_MIN;
        for (int q = 0; q < a.p; ++q) mx = max(mx, ld_relaxed_i32(base + (size_t)q * n_layers + l));
        E_glob[l] = mx;
    }
}

// ------------------------------------------------------------------ signal / wait
__global__ void peer_signal_kernel(PeerArgs a, int slot, int next)
{
    __shared__ uint32_t s_epoch;
    uint32_t *mine = a.flags[a.rank];
    if (threadIdx.x == 0) {
        const uint32_t e = mine[kMineR] + (next ? 1u : 0u);
        mine[kMineR] = e;
        s_epoch = e;
        __threadfence_system();
    }
    __syncthreads();
    for (int q = threadIdx.x; q < a.p; q += blockDim.x) st_release_sys(a.flags[q] + slot + a.rank, s_epoch);
}

__global__ void peer_wait_kernel(PeerArgs a, int slot, uint32_t *err_flag)
{
    if (threadIdx.x == 0) wait_all(a, slot, a.flags[a.rank][kMineR], err_flag);
}

// signal + wait in one launch (real ranks: every rank runs it concurrently; the
// simulated ranks of one device need the two halves as separate launches)
__global__ void peer_signal_wait_kernel(PeerArgs a, int slot, int next, uint32_t *err_flag)
{
    if (threadIdx.x != 0) return;
    uint32_t *mine = a.flags[a.rank];
    const uint32_t e = mine[kMineR] + (next ? 1u : 0u);
    mine[kMineR] = e;
    __threadfence_system();
    for (int q = 0; q < a.p; ++q) st_release_sys(a.flags[q] + slot + a.rank, e);
    wait_all(a, slot, e, err_flag);
}

// post + collect of the E exchange in one launch (real ranks)
__global__ void peer_exchange_E_kernel(PeerArgs a, const int32_t *E_local, int32_t *E_glob, int n_layers,
                                       uint32_t *err_flag)
{
    __shared__ uint32_t s_epoch;
    uint32_t *mine = a.flags[a.rank];
    if (threadIdx.x == 0) s_epoch = mine[kMineE] + 1u;
    __syncthreads();
    const uint32_t epoch = s_epoch;
    const size_t par = (size_t)(epoch & 1u) * (size_t)a.p + (size_t)a.rank;
    for (int q = 0; q < a.p; ++q) {
        int32_t *dst = a.eslots[q] + par * (size_t)n_layers;
        for (int l = threadIdx.x; l < n_layers; l += blockDim.x) dst[l] = E_local[l];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mine[kMineE] = epoch;
        __threadfence_system();
        for (int q = 0; q < a.p; ++q) st_release_sys(a.flags[q] + kSlotE + a.rank, epoch);
        wait_all(a, kSlotE, epoch, err_flag);
    }
    __syncthreads();
    const int32_t *base = a.eslots[a.rank] + (size_t)(epoch & 1u) * (size_t)a.p * (size_t)n_layers;
    for (int l = threadIdx.x; l < n_layers; l += blockDim.x) {
        int32_t mx = INT32_MIN;
        for (int q = 0; q < a.p; ++q) mx = max(mx, ld_relaxed_i32(base + (size_t)q * n_layers + l));
        E_glob[l] = mx;
    }
}

// ------------------------------------------------------------------ the fold
// Reduction schedule of one tile: rank of the j-th addend of group gi.
struct Order {
    int k, G, c1, c2;
    __device__ __forceinline__ Order(const PeerArgs &a, int64_t t)
    {
        k = a.group_k;
        G = a.p / a.group_k;
        // T' < 2^31 tiles (aps_init); 32-bit divisions
        c1 = (int)((uint32_t)t / (uint32_t)(a.tiles / k));
        c2 = (int)((uint32_t)t / (uint32_t)(a.tiles / G));
    }
    __device__ __forceinline__ int rank_of(int gi, int j) const
    {
        int g = c2 + 1 + gi;  // < 2G: one conditional subtraction is the mod
        g = g >= G ? g - G : g;
        int u = c1 + 1 + j;
        u = u >= k ? u - k : u;
        return g * k + u;
    }
};

// Rounding of the accumulator.  EXT = false: the wire format itself (s <- Cast(fl32(s + x)),
// reading A13); EXT = true: the accumulator format A, optionally Kahan-compensated
// (reading A24).  Values are carried as fp32 (every format value is exact in fp32).
template <class C, class A, bool EXT>
__device__ __forceinline__ float rnd(const C &cw, const A &ca, float x)
{
    if constexpr (EXT) return ca.dec(ca.enc(x));
    else return cw.dec(cw.enc(x));
}

template <class C, class A, bool EXT, bool KAHAN>
__device__ __forceinline__ void fold_add(const C &cw, const A &ca, float &s, float &c, float x)
{
    if constexpr (KAHAN) {
        const float y = rnd<C, A, EXT>(cw, ca, __fsub_rn(x, c));
        const float t = rnd<C, A, EXT>(cw, ca, __fadd_rn(s, y));
        c = rnd<C, A, EXT>(cw, ca, __fsub_rn(rnd<C, A, EXT>(cw, ca, __fsub_rn(t, s)), y));
        s = t;
    } else {
        s = rnd<C, A, EXT>(cw, ca, __fadd_rn(s, x));
    }
}

// ------------------------------------------------------------------ fp8 fold in binary16 pairs
// For the hardware fp8 codecs (5,2) / (4,3) with the wire-format accumulator the
// fold runs on f16x2: dec = cvt.rn.f16x2.{e5m2,e4m3}x2 (exact: every fp8 value is a
// binary16), add = add.rn.f16x2, re-quantise = cvt.rn.satfinite.{e5m2,e4m3}x2.f16x2.
// Cast(fl16(a + b)) == Cast(fl32(a + b)) == the exactly rounded sum: binary16
// carries p' = 11 >= 2p + 1 significant bits (p = 3 / 4) in every binade the
// fp8 formats reach, including their subnormals (binary16's ulp there is 2^-24),
// so the double rounding is innocuous (Figueroa), and APS partial sums stay
// <= 1.5 * 2^bias < 65504 (no binary16 overflow) and below the satfinite clamp
// (reading A12).  Exhaustively checked on the device against the oracle
// (tests/test_gpu_peer.py::test_peer_fp8_all_code_pairs).
template <bool E4M3>
__device__ __forceinline__ __half2 fp8x2_to_h2(uint32_t two)
{
    uint32_t h2;
    if (E4M3) asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)two));
    else asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)two));
    return *reinterpret_cast<__half2 *>(&h2);
}
template <bool E4M3>
__device__ __forceinline__ uint32_t h2_to_fp8x2(__half2 h)
{
    uint16_t d;
    const uint32_t v = *reinterpret_cast<uint32_t *>(&h);
    if (E4M3) asm("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;" : "=h"(d) : "r"(v));
    else asm("cvt.rn.satfinite.e5m2x2.f16x2 %0, %1;" : "=h"(d) : "r"(v));
    return d;
}

// e5m2 is binary16 with its low 8 significand bits dropped (same sign, exponent field and
// bias; its subnormals are binary16's with the low byte zero), so on f16x2 words:
//   decode  = move the code byte into the high byte of each half (one byte permute),
//   Cast    = round each half to its high byte, ties to even, on the bit pattern:
//             (u + 0x7f + lsb) & 0xff00 -- the carry runs into the exponent exactly as RNE
//             does, and cannot cross halves (|sum| <= 1.5 * 2^15 < 0x7f80, reading A12),
//   encode  = gather the high bytes (one byte permute),
// all full-rate integer ops instead of the F2FP conversions (compile-time A/B switch).
#ifndef APS_PEER_E5M2_INT
#define APS_PEER_E5M2_INT 0  // measured: 1 (integer fold) 0.28 ms vs 0 (F2FP) 0.265 ms for the simulated p = 8 all-reduce (profiles/r02d_peer_ab.txt)
#endif
template <bool E4M3>
__device__ __forceinline__ __half2 dec_pair(uint32_t w, int hi)
{
    if constexpr (!E4M3 && APS_PEER_E5M2_INT) {
        const uint32_t h = __byte_perm(w, 0u, hi ? 0x3424 : 0x1404);
        return *reinterpret_cast<const __half2 *>(&h);
    } else {
        return fp8x2_to_h2<E4M3>(hi ? (w >> 16) : (w & 0xffffu));
    }
}
template <bool E4M3>
__device__ __forceinline__ __half2 requant_h2(__half2 v)
{
    if constexpr (!E4M3 && APS_PEER_E5M2_INT) {
        const uint32_t u = *reinterpret_cast<const uint32_t *>(&v);
        const uint32_t r = (u + 0x007f007fu + ((u >> 8) & 0x00010001u)) & 0xff00ff00u;
        return *reinterpret_cast<const __half2 *>(&r);
    } else {
        return fp8x2_to_h2<E4M3>(h2_to_fp8x2<E4M3>(v));
    }
}
// two pairs already on the format's grid -> 4 codes
template <bool E4M3>
__device__ __forceinline__ uint32_t enc_pairs(__half2 a, __half2 b)
{
    if constexpr (!E4M3 && APS_PEER_E5M2_INT) {
        return __byte_perm(*reinterpret_cast<const uint32_t *>(&a), *reinterpret_cast<const uint32_t *>(&b), 0x7531);
    } else {
        return h2_to_fp8x2<E4M3>(a) | (h2_to_fp8x2<E4M3>(b) << 16);
    }
}

template <bool E4M3, int NT>
#ifndef APS_PEER_MINB
#define APS_PEER_MINB 3  // measured: 2 -> 19 us, 3 -> 17.2 us, 4 (64 regs, spills) -> 19.5 us (profiles/r01_ab_peer_minblocks.txt)
#endif
__global__ void __launch_bounds__(NT, APS_PEER_MINB) peer_reduce_fp8h_kernel(PeerArgs a, int64_t byte_off, int64_t tile0,
                                                              int64_t n_vec)
{
#ifndef APS_PEER_BATCH
#define APS_PEER_BATCH 8  // addends loaded per batch (registers vs loads in flight; A/B)
#endif
    constexpr int kBatch = APS_PEER_BATCH;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n_vec; i += (int64_t)gridDim.x * NT) {
        const int64_t off = byte_off + i * 16;
        const Order o(a, tile0 + i / 8);  // a tile is 128 bytes = 8 vectors
        __half2 S[8], s[8];               // 16 codes as 8 pairs
        int gi = 0, j = 0;
        for (int idx0 = 0; idx0 < a.p; idx0 += kBatch) {
            uint4 v[kBatch];
            const int nb = min(kBatch, a.p - idx0);
            {
                int g2 = gi, j2 = j;
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (u < nb) v[u] = ld_peer16(a.packed[o.rank_of(g2, j2)] + off);
                    if (++j2 == o.k) {
                        j2 = 0;
                        ++g2;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (u >= nb) break;
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const __half2 x = dec_pair<E4M3>(w[q >> 1], q & 1);
                    s[q] = (j == 0) ? x : requant_h2<E4M3>(__hadd2(s[q], x));
                }
                if (j == o.k - 1) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        S[q] = (gi == 0) ? s[q] : requant_h2<E4M3>(__hadd2(S[q], s[q]));
                    j = 0;
                    ++gi;
                } else {
                    ++j;
                }
            }
        }
        uint4 r;
        r.x = enc_pairs<E4M3>(S[0], S[1]);
        r.y = enc_pairs<E4M3>(S[2], S[3]);
        r.z = enc_pairs<E4M3>(S[4], S[5]);
        r.w = enc_pairs<E4M3>(S[6], S[7]);
        for (int q = 0; q < a.p; ++q) *reinterpret_cast<uint4 *>(a.packed[q] + off) = r;
    }
    cta_fence_system();
}

// ------------------------------------------------------------------ reduce, direct widths (b = 8, 16, 32)
// One 16-byte vector (16 / 8 / 4 codes) per thread and iteration; all codes of
// a vector share a tile, hence one reduction schedule.
template <int B, class C, class A, bool EXT, bool KAHAN, int NT>
__global__ void __launch_bounds__(NT) peer_reduce_direct_kernel(PeerArgs a, int64_t byte_off, int64_t tile0,
                                                                int64_t n_vec, C cw, A ca)
{
    using W = typename Word4<B>::T;
    constexpr int G4 = 16 / sizeof(W);  // 4-code groups per vector
    constexpr int NC = 4 * G4;
    constexpr int kBatch = 8;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n_vec; i += (int64_t)gridDim.x * NT) {
        const int64_t off = byte_off + i * 16;
        const Order o(a, tile0 + (i * 16) / (16 * B));
        // the p addends in fold order (group gi = idx / k, member j = idx % k), loaded
        // kBatch at a time so that many peer loads are in flight per thread
        float S[NC], Sc[NC], s[NC], c[NC];
        int gi = 0, j = 0;
        for (int idx0 = 0; idx0 < a.p; idx0 += kBatch) {
            uint4 v[kBatch];
            const int nb = min(kBatch, a.p - idx0);
            {
                int g2 = gi, j2 = j;
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (u < nb) v[u] = ld_peer16(a.packed[o.rank_of(g2, j2)] + off);
                    if (++j2 == o.k) {
                        j2 = 0;
                        ++g2;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (u >= nb) break;
                W w[G4];
                memcpy(w, &v[u], 16);
#pragma unroll
                for (int g = 0; g < G4; ++g) {
                    const float4 x = unpack4<B>(cw, w[g]);
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int n = 4 * g + h;
                        if (j == 0) {
                            s[n] = EXT ? rnd<C, A, EXT>(cw, ca, xs[h]) : xs[h];
                            c[n] = 0.f;
                        } else {
                            fold_add<C, A, EXT, KAHAN>(cw, ca, s[n], c[n], xs[h]);
                        }
                    }
                }
                if (j == o.k - 1) {  // group complete: fold its sum into the masters' sum
#pragma unroll
                    for (int n = 0; n < NC; ++n) {
                        if (gi == 0) {
                            S[n] = s[n];
                            Sc[n] = 0.f;
                        } else {
                            fold_add<C, A, EXT, KAHAN>(cw, ca, S[n], Sc[n], s[n]);
                        }
                    }
                    j = 0;
                    ++gi;
                } else {
                    ++j;
                }
            }
        }
        W w[G4];
#pragma unroll
        for (int g = 0; g < G4; ++g) w[g] = pack4<B>(cw, make_float4(S[4 * g], S[4 * g + 1], S[4 * g + 2], S[4 * g + 3]));
        uint4 r;
        memcpy(&r, w, 16);
        for (int q = 0; q < a.p; ++q) *reinterpret_cast<uint4 *>(a.packed[q] + off) = r;
    }
    cta_fence_system();
}

// ------------------------------------------------------------------ reduce, any width (per-warp tile)
template <class C, class A, bool EXT, bool KAHAN, int NT>
__global__ void __launch_bounds__(NT) peer_reduce_tile_kernel(PeerArgs a, int64_t byte_off, int64_t tile0,
                                                              int64_t n_tiles, C cw, A ca)
{
    __shared__ __align__(16) uint32_t s_w[NT / 32][kTile + 1];
    const int b = cw.b();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *wa = s_w[warp];
    const int64_t warps = (int64_t)gridDim.x * (NT / 32);
    if (b <= kRegMaxB) {
        // b <= 16: each lane loads the 2-3 words of every rank's tile its bits touch, splits
        // its 4 codes out, folds, and the reduced tile is re-packed in registers
        constexpr int BB = (C::kB > 0 && C::kB <= kRegMaxB) ? C::kB : 0;
        for (int64_t tt = blockIdx.x * (int64_t)(NT / 32) + warp; tt < n_tiles; tt += warps) {
            const int64_t off = byte_off + tt * 16 * b;
            const Order o(a, tile0 + tt);
            float S[4], Sc[4], s[4], c[4];
            for (int gi = 0; gi < o.G; ++gi) {
                for (int j = 0; j < o.k; ++j) {
                    const uint8_t *src = a.packed[o.rank_of(gi, j)] + off;
                    const uint4 cd = tile_split<BB>(
                        tile_fetch<BB>(reinterpret_cast<const uint32_t *>(src), b, lane,
                                       [](const uint32_t *q) { return ld_peer4(q); }),
                        b, lane);
                    const uint32_t cv[4] = {cd.x, cd.y, cd.z, cd.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float x = cw.dec(cv[h]);
                        if (j == 0) {
                            s[h] = EXT ? rnd<C, A, EXT>(cw, ca, x) : x;
                            c[h] = 0.f;
                        } else {
                            fold_add<C, A, EXT, KAHAN>(cw, ca, s[h], c[h], x);
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    if (gi == 0) {
                        S[h] = s[h];
                        Sc[h] = 0.f;
                    } else {
                        fold_add<C, A, EXT, KAHAN>(cw, ca, S[h], Sc[h], s[h]);
                    }
                }
            }
            const TileSlots wo = tile_pack<BB>(make_uint4(cw.enc(S[0]), cw.enc(S[1]), cw.enc(S[2]), cw.enc(S[3])), b, lane);
            for (int q = 0; q < a.p; ++q) {
                uint32_t *tw = reinterpret_cast<uint32_t *>(a.packed[q] + off);
                tile_store(wo, [&](int i, uint32_t x) { tw[i] = x; });
            }
        }
        cta_fence_system();
        return;
    }
    for (int64_t tt = blockIdx.x * (int64_t)(NT / 32) + warp; tt < n_tiles; tt += warps) {
        const int64_t off = byte_off + tt * 16 * b;
        const Order o(a, tile0 + tt);
        float S[4], Sc[4], s[4], c[4];
        for (int gi = 0; gi < o.G; ++gi) {
            for (int j = 0; j < o.k; ++j) {
                const uint8_t *src = a.packed[o.rank_of(gi, j)] + off;
                __syncwarp();
                for (int w = lane; w < 4 * b; w += 32) wa[w] = ld_peer4(src + 4 * w);
                if (lane == 0) wa[4 * b] = 0u;
                __syncwarp();
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float x = cw.dec(extract_code(wa, lane * 4 + h, b));
                    if (j == 0) {
                        s[h] = EXT ? rnd<C, A, EXT>(cw, ca, x) : x;
                        c[h] = 0.f;
                    } else {
                        fold_add<C, A, EXT, KAHAN>(cw, ca, s[h], c[h], x);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (gi == 0) {
                    S[h] = s[h];
                    Sc[h] = 0.f;
                } else {
                    fold_add<C, A, EXT, KAHAN>(cw, ca, S[h], Sc[h], s[h]);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 4; ++h) wa[lane * 4 + h] = cw.enc(S[h]);
        __syncwarp();
        for (int w = lane; w < 4 * b; w += 32) {
            const uint32_t word = assemble_word(wa, w, b);
            for (int q = 0; q < a.p; ++q) reinterpret_cast<uint32_t *>(a.packed[q] + off)[w] = word;
        }
    }
    cta_fence_system();
}

// ------------------------------------------------------------------ stochastic rounding (reading A26)
// r = SplitMix64(seed, phase << 40 | i) >> 32 (the same counter-based generator the
// oracle implements); x between its neighbours lo <= |x| < hi rounds up iff
// r < (|x| - lo) / (hi - lo) * 2^32.  Phase: rank for the Cast of a rank's gradient,
// p - 1 + a for the a-th add of an element's fold.
__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t ctr)
{
    uint64_t z = seed + (ctr + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t sr_rand(uint64_t seed, uint64_t phase, int64_t i)
{
    return (uint32_t)(splitmix64(seed, (phase << 40) | (uint64_t)i) >> 32);
}
// per-call key (reading A27): the k-th sync after aps_set_rounding(seed) draws with
// seed_k = SplitMix64(seed, k); k is the device-resident call counter (capture-safe)
__device__ __forceinline__ uint64_t sr_call_seed(uint64_t seed, const uint32_t *call)
{
    return splitmix64(seed, (uint64_t)*call);
}

__global__ void sr_advance_kernel(uint32_t *call) { ++*call; }

// up iff r < rem / 2^d * 2^32 (exact, any d >= 1)
__device__ __forceinline__ uint32_t sr_up(uint32_t r, uint64_t rem, int d)
{
    if (rem == 0) return 0u;
    if (d <= 32) return (uint32_t)((r >> (32 - d)) < rem);
    if (d - 32 >= 24) return (uint32_t)(r == 0u);         // rem < 2^24 <= 2^(d-32)
    return (uint32_t)(((uint64_t)r << (d - 32)) < rem);
}

__device__ __forceinline__ uint32_t encode_sr(const Fmt &F, float y, uint32_t r)
{
    const uint32_t u = __float_as_uint(y);
    const uint32_t a = u & 0x7fffffffu;
    const uint32_t s = (u >> 31) << (F.e + F.m);
    if (a > 0x7f800000u) return s | F.nan_code;
    if (a == 0u) return s;
    if (F.m == 23) return u;                                          // (8,23): identity
    const uint32_t inf_bits = (uint32_t)(127 + F.bias + 1) << 23;     // 2^(bias+1)
    if (a >= inf_bits) return s | F.inf_code;
    uint32_t mag;
    if (a >= F.norm_min) {                                            // target normal: d = 23 - m
        mag = (a >> F.sh) - F.rebias + sr_up(r, a & ((1u << F.sh) - 1u), (int)F.sh);
    } else {                                                          // target subnormal
        const uint64_t sig = (a >= 0x800000u) ? ((a & 0x7fffffu) | 0x800000u) : a;
        const int lsb = (a >= 0x800000u) ? (int)(a >> 23) - 150 : -149;
        const int d = (1 - F.bias - F.m) - lsb;
        if (d <= 0) {
            mag = (uint32_t)(sig << (-d));
        } else {
            const uint64_t n = d >= 64 ? 0ull : (sig >> d);
            const uint64_t rem = d >= 64 ? sig : (sig & ((1ull << d) - 1ull));
            mag = (uint32_t)n + sr_up(r, rem, d);
        }
    }
    return s | min(mag, F.inf_code);
}

// a3+a4 with stochastic rounding, any width: per warp one tile of 128 codes
template <int NT>
__global__ void __launch_bounds__(NT) quant_pack_sr_kernel(DevTables t, Fmt F, uint64_t seed0, int rank)
{
    const uint64_t seed = sr_call_seed(seed0, t.sr_call);
    __shared__ __align__(16) uint32_t s_codes[NT / 32][kTile + 1];
    const Item it = t.items[blockIdx.x];
    const LayerDev L = t.layers[it.layer];
    const float *g = t.src[it.layer];
    const int ft = scale_exponent(t, it.layer, F.bias, it.tile_begin == 0 && threadIdx.x == 0);
    const Pow2 sc(ft);
    const int b = F.b;
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    const int64_t n = min((int64_t)it.n_tiles * kTile, L.numel - begin);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *codes = s_codes[warp];
    uint32_t *out = reinterpret_cast<uint32_t *>(t.packed + it.byte_pos);
    for (int tt = warp; tt < it.n_tiles; tt += NT / 32) {
        const int64_t e0 = (int64_t)tt * kTile + lane * 4;
        const float4 y = sc.apply4(load_group(g + begin, e0, n));
        const int64_t idx = (it.tile_pos + tt) * kTile + lane * 4;  // code index in the packed layout
        const float ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) codes[lane * 4 + h] = encode_sr(F, ys[h], sr_rand(seed, (uint64_t)rank, idx + h));
        __syncwarp();
        uint32_t *ow = out + (int64_t)tt * (4 * b);
        for (int w = lane; w < 4 * b; w += 32) ow[w] = assemble_word(codes, w, b);
        __syncwarp();
    }
}

// owner-computes reduce with a stochastic re-quantise after every add (wire accumulator)
template <int NT>
__global__ void __launch_bounds__(NT) peer_reduce_sr_kernel(PeerArgs a, int64_t byte_off, int64_t tile0,
                                                            int64_t n_tiles, Fmt F, uint64_t seed0, const uint32_t *call)
{
    const uint64_t seed = sr_call_seed(seed0, call);
    __shared__ __align__(16) uint32_t s_w[NT / 32][kTile + 1];
    const int b = F.b;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *wa = s_w[warp];
    const int64_t warps = (int64_t)gridDim.x * (NT / 32);
    for (int64_t tt = blockIdx.x * (int64_t)(NT / 32) + warp; tt < n_tiles; tt += warps) {
        const int64_t off = byte_off + tt * 16 * b;
        const int64_t t = tile0 + tt;
        const Order o(a, t);
        float S[4], s[4];
        int adds = 0;
        for (int gi = 0; gi < o.G; ++gi) {
            for (int j = 0; j < o.k; ++j) {
                const uint8_t *src = a.packed[o.rank_of(gi, j)] + off;
                __syncwarp();
                for (int w = lane; w < 4 * b; w += 32) wa[w] = ld_peer4(src + 4 * w);
                if (lane == 0) wa[4 * b] = 0u;
                __syncwarp();
                if (j > 0) ++adds;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float x = decode_finite(F, extract_code(wa, lane * 4 + h, b));
                    const int64_t idx = t * kTile + lane * 4 + h;
                    s[h] = (j == 0) ? x
                                    : decode_finite(F, encode_sr(F, __fadd_rn(s[h], x),
                                                                 sr_rand(seed, (uint64_t)(a.p - 1 + adds), idx)));
                }
            }
            if (gi > 0) ++adds;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int64_t idx = t * kTile + lane * 4 + h;
                S[h] = (gi == 0) ? s[h]
                                 : decode_finite(F, encode_sr(F, __fadd_rn(S[h], s[h]),
                                                              sr_rand(seed, (uint64_t)(a.p - 1 + adds), idx)));
            }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 4; ++h) wa[lane * 4 + h] = encode(F, S[h]);
        __syncwarp();
        for (int w = lane; w < 4 * b; w += 32) {
            const uint32_t word = assemble_word(wa, w, b);
            for (int q = 0; q < a.p; ++q) reinterpret_cast<uint32_t *>(a.packed[q] + off)[w] = word;
        }
    }
    cta_fence_system();
}

__global__ void debug_cast_sr_kernel(const float *in, uint32_t *codes, int64_t n, Fmt F, uint64_t seed, uint64_t phase)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        codes[i] = encode_sr(F, in[i], sr_rand(seed, phase, i));
}

cudaError_t launch_debug_cast_sr(const float *in, uint32_t *codes, int64_t n, int e, int m, uint64_t seed,
                                 uint64_t phase, cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
    debug_cast_sr_kernel<<<grid, 256, 0, s>>>(in, codes, n, make_fmt(e, m), seed, phase);
    return cudaGetLastError();
}

cudaError_t launch_quant_pack_sr(const DevTables &t, int e, int m, uint64_t seed, int rank, cudaStream_t s)
{
    if (t.n_items == 0) return cudaSuccess;
    quant_pack_sr_kernel<kThreads><<<t.n_items, kThreads, 0, s>>>(t, make_fmt(e, m), seed, rank);
    return cudaGetLastError();
}

cudaError_t launch_peer_reduce_sr(const PeerArgs &a, int64_t byte_off, int64_t tile0, int64_t n_tiles, int e, int m,
                                  uint64_t seed, const uint32_t *call, cudaStream_t s)
{
    if (n_tiles <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n_tiles + kThreads / 32 - 1) / (kThreads / 32), (int64_t)sm_count() * 8);
    peer_reduce_sr_kernel<kThreads><<<grid, kThreads, 0, s>>>(a, byte_off, tile0, n_tiles, make_fmt(e, m), seed, call);
    return cudaGetLastError();
}

cudaError_t launch_sr_advance(uint32_t *call, cudaStream_t s)
{
    sr_advance_kernel<<<1, 1, 0, s>>>(call);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_peer_post_E(const PeerArgs &a, const int32_t *E_local, int n_layers, cudaStream_t s)
{
    peer_post_E_kernel<<<1, 1024, 0, s>>>(a, E_local, n_layers);
    return cudaGetLastError();
}

cudaError_t launch_peer_collect_E(const PeerArgs &a, int32_t *E_glob, int n_layers, uint32_t *err_flag,
                                  cudaStream_t s)
{
    peer_collect_E_kernel<<<1, 1024, 0, s>>>(a, E_glob, n_layers, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_peer_signal(const PeerArgs &a, int slot, bool next, cudaStream_t s)
{
    peer_signal_kernel<<<1, 64, 0, s>>>(a, slot, next ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_peer_signal_wait(const PeerArgs &a, int slot, bool next, uint32_t *err_flag, cudaStream_t s)
{
    peer_signal_wait_kernel<<<1, 32, 0, s>>>(a, slot, next ? 1 : 0, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_peer_exchange_E(const PeerArgs &a, const int32_t *E_local, int32_t *E_glob, int n_layers,
                                   uint32_t *err_flag, cudaStream_t s)
{
    peer_exchange_E_kernel<<<1, 1024, 0, s>>>(a, E_local, E_glob, n_layers, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_peer_wait(const PeerArgs &a, int slot, uint32_t *err_flag, cudaStream_t s)
{
    peer_wait_kernel<<<1, 32, 0, s>>>(a, slot, err_flag);
    return cudaGetLastError();
}

template <class C, class A, bool EXT, bool KAHAN>
static cudaError_t launch_reduce_t(const PeerArgs &a, int64_t byte_off, int64_t tile0, int64_t n_tiles, int b, C cw,
                                   A ca, cudaStream_t s)
{
    const int64_t n_vec = n_tiles * b;  // a tile is 16 b bytes = b vectors
    // one resident wave (2 CTAs of 256 threads per SM at ~96 registers): every CTA
    // pays its closing system fence once
    const int grid_direct = (int)std::min<int64_t>((n_vec + kThreads - 1) / kThreads, (int64_t)sm_count() * 2);
    const int grid_tile =
        (int)std::min<int64_t>((n_tiles + kThreads / 32 - 1) / (kThreads / 32), (int64_t)sm_count() * 8);
    if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32) {
        peer_reduce_direct_kernel<C::kB, C, A, EXT, KAHAN, kThreads><<<grid_direct, kThreads, 0, s>>>(
            a, byte_off, tile0, n_vec, cw, ca);
    } else if constexpr (C::kB == 0) {
        if (b == 8)
            peer_reduce_direct_kernel<8, C, A, EXT, KAHAN, kThreads><<<grid_direct, kThreads, 0, s>>>(a, byte_off, tile0,
                                                                                                     n_vec, cw, ca);
        else if (b == 16)
            peer_reduce_direct_kernel<16, C, A, EXT, KAHAN, kThreads><<<grid_direct, kThreads, 0, s>>>(a, byte_off, tile0,
                                                                                                      n_vec, cw, ca);
        else if (b == 32)
            peer_reduce_direct_kernel<32, C, A, EXT, KAHAN, kThreads><<<grid_direct, kThreads, 0, s>>>(a, byte_off, tile0,
                                                                                                      n_vec, cw, ca);
        else
            peer_reduce_tile_kernel<C, A, EXT, KAHAN, kThreads><<<grid_tile, kThreads, 0, s>>>(a, byte_off, tile0,
                                                                                              n_tiles, cw, ca);
    } else {
        peer_reduce_tile_kernel<C, A, EXT, KAHAN, kThreads><<<grid_tile, kThreads, 0, s>>>(a, byte_off, tile0, n_tiles,
                                                                                          cw, ca);
    }
    return cudaGetLastError();
}

cudaError_t launch_peer_reduce(const PeerArgs &a, int64_t byte_off, int64_t tile0, int64_t n_tiles, int e, int m,
                               bool hw, int acc_e, int acc_m, bool kahan, cudaStream_t s)
{
    if (n_tiles <= 0) return cudaSuccess;
    const int b = 1 + e + m;
    const bool ext = kahan || acc_e != e || acc_m != m;
    if (!ext && hw && ((e == 5 && m == 2) || (e == 4 && m == 3))) {
        const int64_t n_vec = n_tiles * 8;
        const int grid = (int)std::min<int64_t>((n_vec + kThreads - 1) / kThreads, (int64_t)sm_count() * APS_PEER_MINB);
        if (e == 5) peer_reduce_fp8h_kernel<false, kThreads><<<grid, kThreads, 0, s>>>(a, byte_off, tile0, n_vec);
        else peer_reduce_fp8h_kernel<true, kThreads><<<grid, kThreads, 0, s>>>(a, byte_off, tile0, n_vec);
        return cudaGetLastError();
    }
    if (!ext)
        return with_codec(e, m, hw, [&](auto cw) -> cudaError_t {
            using C = decltype(cw);
            return launch_reduce_t<C, C, false, false>(a, byte_off, tile0, n_tiles, b, cw, cw, s);
        });
    // accumulator variants (off the headline path): runtime wire codec (bit-identical
    // to the specialised ones), binary32 or runtime accumulator codec
    CRt cw;
    cw.F = make_fmt(e, m);
    if (acc_e == 8 && acc_m == 23) {  // binary32 accumulator: rounding is the identity
        if (kahan) return launch_reduce_t<CRt, CF32, true, true>(a, byte_off, tile0, n_tiles, b, cw, CF32{}, s);
        return launch_reduce_t<CRt, CF32, true, false>(a, byte_off, tile0, n_tiles, b, cw, CF32{}, s);
    }
    CRt ca;
    ca.F = make_fmt(acc_e, acc_m);
    if (kahan) return launch_reduce_t<CRt, CRt, true, true>(a, byte_off, tile0, n_tiles, b, cw, ca, s);
    return launch_reduce_t<CRt, CRt, true, false>(a, byte_off, tile0, n_tiles, b, cw, ca, s);
}

// ------------------------------------------------------------------ Eq. (5) round-off metric
// sum over i with h_i != 0 of |(h_i - l_i) / h_i| (binary64) and the count of such i.
__global__ void round_off_kernel(const float *h, const float *l, int64_t n, double *sum, unsigned long long *cnt)
{
    double acc = 0.0;
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float hv = h[i];
        if (hv != 0.f) {
            acc += fabs(((double)hv - (double)l[i]) / (double)hv);
            ++c;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    __shared__ double s_acc[32];
    __shared__ unsigned long long s_c[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_acc[warp] = acc;
        s_c[warp] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            acc += s_acc[w];
            c += s_c[w];
        }
        atomicAdd(sum, acc);
        atomicAdd(cnt, c);
    }
}

// ------------------------------------------------------------------ underflow / overflow census
// One CTA per work item: counts the nonzero finite elements whose Cast(g * 2^s_l)
// (generic codec: IEEE overflow to Inf, never the saturating hardware converter)
// is +-0 (underflow) or +-Inf (overflow); counts[2 l], counts[2 l + 1].
template <int NT>
__global__ void __launch_bounds__(NT) census_kernel(DevTables t, const int32_t *sexp, unsigned long long *counts,
                                                    Fmt F)
{
    const Item it = t.items[blockIdx.x];
    const float *g = t.src[it.layer] + (int64_t)it.tile_begin * kTile;
    const Pow2 sc(sexp[it.layer]);
    const uint32_t inf_mag = F.inf_code;
    unsigned long long u = 0, o = 0;
    for (int i = threadIdx.x; i < it.cnt; i += NT) {
        const float x = g[i];
        if (x == 0.f || !isfinite(x)) continue;
        const uint32_t mag = encode(F, sc.apply(x)) & F.mag_mask;
        u += (mag == 0u);
        o += (mag == inf_mag);
    }
    u = __reduce_add_sync(0xffffffffu, (uint32_t)u);
    o = __reduce_add_sync(0xffffffffu, (uint32_t)o);
    if ((threadIdx.x & 31) == 0) {
        if (u) atomicAdd(&counts[2 * it.layer], u);
        if (o) atomicAdd(&counts[2 * it.layer + 1], o);
    }
}

cudaError_t launch_census(const DevTables &t, const int32_t *sexp, unsigned long long *counts, int e, int m,
                          cudaStream_t s)
{
    if (t.n_items == 0) return cudaSuccess;
    census_kernel<kThreads><<<t.n_items, kThreads, 0, s>>>(t, sexp, counts, make_fmt(e, m));
    return cudaGetLastError();
}

cudaError_t launch_round_off(const float *h, const float *l, int64_t n, double *sum, unsigned long long *cnt,
                             cudaStream_t s)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n + 1023) / 1024, (int64_t)sm_count() * 4);
    round_off_kernel<<<grid, 1024, 0, s>>>(h, l, n, sum, cnt);
    return cudaGetLastError();
}

}  // namespace aps
