// aps_stream.cu -- persistent, TMA-bulk pipelined versions of the HBM-bound
// APS kernels for sm_100a.
//
// Every hot kernel of the path streams each gradient element through the SM
// once per pass, so it is bound by HBM bandwidth, and short (~20 us at
// ResNet-50 size): CTA launch ramp and tail matter as much as steady-state
// bandwidth.  The engine runs ONE persistent CTA per SM:
//
//   producer (warp 8): its 32 lanes prefetch the flat descriptors (and side
//     information: layer pointers, f~) of the CTA's next 32 work items in
//     parallel; lane 0 then, per item, waits for a free stage, arms the
//     stage's `full` mbarrier with the byte count and issues ONE
//     cp.async.bulk global->shared copy of up to 32 KB (the TMA bulk engine
//     sustains ~7 TB/s chip-wide only with >= 16-32 KB requests:
//     profiles/r01_microbench_stream.txt), with an L2 eviction-priority
//     hint.  `full` needs two arrivals: the load's, and "side info final".
//   consumers (warps 0..7): wait `full`, each warp transforms a contiguous
//     1024-element chunk in shared memory (results in place or into the
//     stage's code area), writes it back with one cp.async.bulk
//     shared->global store, waits until the stage has been read, and frees
//     it (`empty`).
// FindMaxExp needs no per-item fence or returning atomic: each warp folds its
// chunk's abs-max into the layer with a fire-and-forget red.max, and each CTA
// publishes "my abs-max pass is done" once (fence + one counter add).
//
// Fused p = 1 path (launch_stream_fused_p1): with one rank there is no
// collective between FindMaxExp and Cast, so a single launch does
//   phase A  abs-max of every work item (forward order; L2 evict_last);
//   phase B  per item, in REVERSE order: scale, Cast, pack (codes -> packed
//            buffer) and Cast back, unscale, average (fp32 -> output).
// The producer issues phase-B loads immediately (the gradients are read-
// only) and supplies f~ -- the second `full` arrival -- once every CTA has
// finished phase A (acquire on the counter).  Reverse order makes the second
// read of the gradients hit the data phase A left in the 126 MB L2 most
// recently.  Phase-A items never wait, so with a co-resident grid
// (cooperative launch) the waits cannot deadlock.  The abs-max accumulators
// are double-buffered by call parity (buffer g&1 in use, buffer (g+1)&1
// cleared for the next call), so no extra pass resets them.
#include <cstdint>
#include <algorithm>
#include <climits>

#include "aps_device.cuh"

namespace aps {

constexpr int kF32Bytes = kItemTiles * kTile * 4;  // 32 KB: one work item of fp32
constexpr int kConsWarps = 8;
constexpr int kConsThreads = kConsWarps * 32;
constexpr int kChunk = kItemTiles * kTile / kConsWarps;  // 1024 elements per consumer warp
constexpr int kStreamThreads = kConsThreads + 32;
constexpr int kSmemBudget = 200 * 1024;

template <int CodeBytes>
struct StageCfg {
    static constexpr int kStageBytes = kF32Bytes + CodeBytes;
    static constexpr int kStages = std::min(6, kSmemBudget / kStageBytes);
};

// Everything the consumers need about a work item, resolved by the
// producer (no consumer touches a global table).
struct StageInfo {
    const float *src;     // gradient at the item's first element
    float *dst;           // output at the item's first element
    int64_t tile_pos;     // first tile of the item in the packed buffer
    int64_t byte_pos;     // its byte offset
    int32_t cnt;          // valid elements
    int32_t n_tiles;
    int32_t layer;
    int32_t first;        // the item holds the layer's first tile
    int32_t ft;           // f~ of the layer (quantise paths)
    int32_t phase_b;      // fused: a quantise item (needs f~ from the finished abs-max)
    int32_t ft_ok;        // ft is final
};

template <int Stages, int StageBytes>
struct StreamSmem {
    alignas(1024) uint8_t stage[Stages][StageBytes];
    uint32_t scratch[kConsWarps][kTile];  // per-warp code tile (generic widths)
    uint64_t full[Stages], empty[Stages];
    StageInfo info[Stages];
    StageInfo batch[32];  // producer: prefetched descriptors of the next 32 items
    int32_t flag;
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// TMA bulk copy shared -> global (bulk async-group completion).
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Load {
    const void *src;
    uint32_t bytes;     // multiple of 16
    uint32_t dst_off;   // byte offset within the stage
    bool keep;          // L2 evict_last (data will be read again) vs evict_first
};

__device__ __forceinline__ void red_max_u32(uint32_t *p, uint32_t v)
{
    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v)
{
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void bar_consumers()
{
    asm volatile("bar.sync 1, %0;" ::"n"(kConsThreads) : "memory");
}

// ------------------------------------------------------------------ item helpers
// Producer-side descriptor fetch (one lane per item, 32 items at a time).
__device__ __forceinline__ StageInfo fetch_info(const DevTables &t, int k, bool want_dst)
{
    const Item it = t.items[k];
    StageInfo si;
    si.layer = it.layer;
    si.cnt = it.cnt;
    si.n_tiles = it.n_tiles;
    si.tile_pos = it.tile_pos;
    si.byte_pos = it.byte_pos;
    si.first = it.tile_begin == 0;
    const int64_t begin = (int64_t)it.tile_begin * kTile;
    si.src = t.src[it.layer] + begin;
    si.dst = want_dst ? t.dst[it.layer] + begin : nullptr;
    si.ft = 0;
    si.phase_b = 0;
    si.ft_ok = 1;
    return si;
}

__device__ __forceinline__ Load grad_load(const StageInfo &si, bool keep)
{
    return Load{si.src, (uint32_t)(si.cnt >> 2) * 16u, 0u, keep};
}

// f~ = upper_bound_exp - E (Alg. 1 line 4) for the layer; the item holding
// the layer's first tile records ftilde[] and the non-finite flag.
__device__ __forceinline__ int ft_from_E(const DevTables &t, int32_t E, int layer, bool first, int bias)
{
    int ft = (E == INT32_MIN) ? 0 : bias - E;
    if (E == INT32_MAX) {
        ft = 0;
        if (first) atomicOr(t.flag, 1u);
    }
    if (first) t.ftilde[layer] = ft;
    return ft;
}

// fp32 group j (elements 4j..4j+3) of an item: from the stage when it was
// bulk-copied, else (the < 4-element tail of a layer) from global memory.
__device__ __forceinline__ float4 stage_group(const float4 *s4, const float *g, int j, int cnt)
{
    if (4 * j + 4 <= cnt) return s4[j];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int e0 = 4 * j;
    if (e0 + 0 < cnt) v.x = g[e0 + 0];
    if (e0 + 1 < cnt) v.y = g[e0 + 1];
    if (e0 + 2 < cnt) v.z = g[e0 + 2];
    return v;
}

// Store the warp's chunk of fp32 results (in the stage) to out[], the < 4
// element tail with plain stores.  elems0: first element of the chunk.
__device__ __forceinline__ void store_chunk_f32(float *out, const float4 *s4, int elems0, int cnt, int lane)
{
    const int n = min(kChunk, cnt - elems0);
    if (n <= 0) return;
    const int n16 = n & ~3;
    if (lane == 0 && n16) bulk_s2g(out + elems0, s4 + elems0 / 4, (uint32_t)n16 * 4u);
    if (lane < (n & 3)) {
        const float *sf = reinterpret_cast<const float *>(s4);
        out[elems0 + n16 + lane] = sf[elems0 + n16 + lane];
    }
}

// a1, consumer side: the warp's abs-max over its chunk, folded into the
// layer's accumulator with a fire-and-forget red.max (bits of |x| are
// monotone in |x|: order-independent, bit-exact).
__device__ __forceinline__ void absmax_chunk(const StageInfo &si, const float4 *s4, uint32_t *amax, int warp,
                                             int lane)
{
    uint32_t mx = 0;
    const int g0 = warp * (kChunk / 4);
    const int n4 = si.cnt >> 2;
#pragma unroll
    for (int k = 0; k < kChunk / 4 / 32; ++k) {
        const int j = g0 + lane + 32 * k;
        if (j < n4) mx = max(mx, absbits4(s4[j]));
    }
    if (warp == kConsWarps - 1 && lane < (si.cnt & 3))
        mx = max(mx, __float_as_uint(si.src[4 * n4 + lane]) & 0x7fffffffu);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0 && mx != 0u) red_max_u32(&amax[si.layer], mx);  // (0 never raises the max)
}

// a3/a4 (+ a7 when Fuse), consumer side, for the warp's chunk.  Codes go to
// `codes` (the stage's code area) and are bulk-stored to the packed buffer;
// with Fuse the unscaled fp32 result overwrites the stage in place and is
// bulk-stored to the output.
template <class C, bool Fuse>
__device__ __forceinline__ void quant_chunk(const DevTables &t, const C &c, const StageInfo &si, uint8_t *stage,
                                            uint8_t *codes, uint32_t *scratch, int avg, int warp, int lane)
{
    constexpr int B = C::kB;
    float4 *s4 = reinterpret_cast<float4 *>(stage);
    const Pow2 s(si.ft);
    const Unscale us(si.ft, 1, avg);
    const int g0 = warp * (kChunk / 4);
    const int tiles_w = min(kChunk / kTile, si.n_tiles - warp * (kChunk / kTile));  // tiles in this chunk
    if (tiles_w <= 0) return;
    if constexpr (B == 8 || B == 16 || B == 32) {
        using W = typename Word4<B>::T;
        W *cw = reinterpret_cast<W *>(codes);
        const int ng = si.n_tiles * (kTile / 4);
        if (!s.wide) {
#pragma unroll
            for (int k = 0; k < kChunk / 4 / 32; ++k) {
                const int j = g0 + lane + 32 * k;
                if (j < ng) {
                    const float4 x = stage_group(s4, si.src, j, si.cnt);
                    const float4 y = make_float4(__fmul_rn(x.x, s.f), __fmul_rn(x.y, s.f), __fmul_rn(x.z, s.f),
                                                 __fmul_rn(x.w, s.f));
                    const W code = pack4<B>(c, y);
                    cw[j] = code;
                    if (Fuse) s4[j] = us.apply4(unpack4<B>(c, code));
                }
            }
        } else {
            for (int k = 0; k < kChunk / 4 / 32; ++k) {
                const int j = g0 + lane + 32 * k;
                if (j < ng) {
                    const W code = pack4<B>(c, s.apply4(stage_group(s4, si.src, j, si.cnt)));
                    cw[j] = code;
                    if (Fuse) s4[j] = us.apply4(unpack4<B>(c, code));
                }
            }
        }
    } else {
        const int b = B;
        uint32_t *cw = reinterpret_cast<uint32_t *>(codes);
        for (int tt = 0; tt < tiles_w; ++tt) {
            const int j = g0 + tt * (kTile / 4) + lane;
            const float4 y = s.apply4(stage_group(s4, si.src, j, si.cnt));
            const uint4 cd = make_uint4(c.enc(y.x), c.enc(y.y), c.enc(y.z), c.enc(y.w));
            __syncwarp();
            *reinterpret_cast<uint4 *>(scratch + 4 * lane) = cd;
            if (Fuse) s4[j] = us.apply4(make_float4(c.dec(cd.x), c.dec(cd.y), c.dec(cd.z), c.dec(cd.w)));
            __syncwarp();
            uint32_t *ow = cw + (int64_t)(warp * (kChunk / kTile) + tt) * (4 * b);
            for (int w = lane; w < 4 * b; w += 32) ow[w] = assemble_word(scratch, w, b);
        }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0)
        bulk_s2g(t.packed + si.byte_pos + (int64_t)warp * (kChunk / kTile) * (16 * B),
                 codes + (size_t)warp * (kChunk / kTile) * (16 * B),
                 (uint32_t)(tiles_w * 16 * B));
    if (Fuse) store_chunk_f32(si.dst, s4, warp * kChunk, si.cnt, lane);
}

// a7, consumer side, for the warp's chunk: codes (loaded into the stage's
// code area) -> fp32 in the stage -> bulk store.
template <class C>
__device__ __forceinline__ void unpack_chunk(const C &c, const StageInfo &si, uint8_t *stage, const uint8_t *codes,
                                             int N, int avg, int warp, int lane)
{
    constexpr int B = C::kB;
    float4 *s4 = reinterpret_cast<float4 *>(stage);
    const Unscale us(si.ft, N, avg);
    const int g0 = warp * (kChunk / 4);
    const int tiles_w = min(kChunk / kTile, si.n_tiles - warp * (kChunk / kTile));
    if (tiles_w <= 0) return;
    if constexpr (B == 8 || B == 16 || B == 32) {
        using W = typename Word4<B>::T;
        const W *cw = reinterpret_cast<const W *>(codes);
        const int ng = si.n_tiles * (kTile / 4);
#pragma unroll
        for (int k = 0; k < kChunk / 4 / 32; ++k) {
            const int j = g0 + lane + 32 * k;
            if (j < ng) s4[j] = us.apply4(unpack4<B>(c, cw[j]));
        }
    } else {
        const int b = B;
        const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes);
        for (int tt = 0; tt < tiles_w; ++tt) {
            const uint32_t *words = cw + (int64_t)(warp * (kChunk / kTile) + tt) * (4 * b);  // words[4b]: masked
            const int k0 = lane * 4;
            const float4 d = make_float4(c.dec(extract_code(words, k0, b)), c.dec(extract_code(words, k0 + 1, b)),
                                         c.dec(extract_code(words, k0 + 2, b)), c.dec(extract_code(words, k0 + 3, b)));
            s4[g0 + tt * (kTile / 4) + lane] = us.apply4(d);
        }
    }
    fence_proxy_async_smem();
    __syncwarp();
    store_chunk_f32(si.dst, s4, warp * kChunk, si.cnt, lane);
}

// ------------------------------------------------------------------ ops
// An Op provides
//   kCodeBytes               size of the stage's code area
//   n_work(), n_phase_a()    work items, and how many of them are abs-max items (first)
//   fetch(w, ready)          producer lane: descriptor and side info of item w
//                            (f~ only when `ready`, i.e. the abs-max pass is complete)
//   late_ft(si)              producer lane: f~ of a phase-B item once ready
//   load(w, si)              the TMA load of item w
//   consume(...)             consumer warp's share of item w
//   absmax buffer, the done-counter target and whether phase B waits on it.
struct AbsmaxOp {
    static constexpr int kCodeBytes = 0;
    DevTables t;
    uint32_t *amax;  // accumulator buffer of this call
    uint32_t *amax_other;
    uint32_t target;
    int N;
    __device__ int n_work() const { return t.n_items; }
    __device__ int n_phase_a() const { return t.n_items; }
    __device__ bool waits() const { return false; }
    __device__ StageInfo fetch(int w, bool) const { return fetch_info(t, w, false); }
    __device__ int late_ft(const StageInfo &) const { return 0; }
    __device__ Load load(int, const StageInfo &si) const { return grad_load(si, true); }
    __device__ void consume(int, uint8_t *stage, const StageInfo &si, uint32_t *, int warp, int lane) const
    {
        absmax_chunk(si, reinterpret_cast<const float4 *>(stage), amax, warp, lane);
    }
    // the last CTA to finish turns the accumulators into E and clears both buffers
    __device__ void after_phase_a_last(int tid) const
    {
        for (int l = tid; l < t.n_layers; l += kConsThreads) {
            t.E_local[l] = exponent_of(amax[l], N);
            amax[l] = 0u;
            amax_other[l] = 0u;
        }
    }
};

template <class C>
struct QuantOp {
    static constexpr int kCodeBytes = kItemTiles * 16 * C::kB;
    DevTables t;
    C c;
    int bias;
    // reverse order: the items a1 read last are still in L2
    __device__ int n_work() const { return t.n_items; }
    __device__ int n_phase_a() const { return 0; }
    __device__ bool waits() const { return false; }
    __device__ StageInfo fetch(int w, bool) const
    {
        StageInfo si = fetch_info(t, t.n_items - 1 - w, false);
        si.ft = ft_from_E(t, t.E_glob[si.layer], si.layer, si.first, bias);
        return si;
    }
    __device__ int late_ft(const StageInfo &si) const { return si.ft; }
    __device__ Load load(int, const StageInfo &si) const { return grad_load(si, false); }
    __device__ void consume(int, uint8_t *stage, const StageInfo &si, uint32_t *scratch, int warp, int lane) const
    {
        quant_chunk<C, false>(t, c, si, stage, stage + kF32Bytes, scratch, 0, warp, lane);
    }
    __device__ void after_phase_a_last(int) const {}
};

template <class C>
struct UnpackOp {
    static constexpr int kCodeBytes = kItemTiles * 16 * C::kB;
    DevTables t;
    C c;
    int N, avg;
    __device__ int n_work() const { return t.n_items; }
    __device__ int n_phase_a() const { return 0; }
    __device__ bool waits() const { return false; }
    __device__ StageInfo fetch(int w, bool) const
    {
        StageInfo si = fetch_info(t, w, true);
        si.ft = t.ftilde[si.layer];
        return si;
    }
    __device__ int late_ft(const StageInfo &si) const { return si.ft; }
    __device__ Load load(int, const StageInfo &si) const
    {
        return Load{t.packed + si.byte_pos, (uint32_t)(16 * C::kB * si.n_tiles), (uint32_t)kF32Bytes,
                    false};
    }
    __device__ void consume(int, uint8_t *stage, const StageInfo &si, uint32_t *, int warp, int lane) const
    {
        unpack_chunk<C>(c, si, stage, stage + kF32Bytes, N, avg, warp, lane);
    }
    __device__ void after_phase_a_last(int) const {}
};

template <class C>
struct FusedP1Op {
    static constexpr int kCodeBytes = kItemTiles * 16 * C::kB;
    DevTables t;
    C c;
    uint32_t *amax;        // accumulator buffer of this call (parity g & 1)
    uint32_t *amax_next;   // the other buffer, cleared here for the next call
    uint32_t target;
    int bias, avg;
    __device__ int n_work() const { return 2 * t.n_items; }
    __device__ int n_phase_a() const { return t.n_items; }
    __device__ bool waits() const { return true; }
    __device__ StageInfo fetch(int w, bool ready) const
    {
        if (w < t.n_items) return fetch_info(t, w, false);
        StageInfo si = fetch_info(t, 2 * t.n_items - 1 - w, true);
        si.phase_b = 1;
        si.ft_ok = ready;
        if (ready) si.ft = late_ft(si);
        return si;
    }
    // E_l from the finished abs-max (N = 1); the layer's first item also
    // records E and clears the other parity buffer.
    __device__ int late_ft(const StageInfo &si) const
    {
        const int32_t E = exponent_of(amax[si.layer], 1);
        if (si.first) {
            t.E_local[si.layer] = E;
            amax_next[si.layer] = 0u;
        }
        return ft_from_E(t, E, si.layer, si.first, bias);
    }
    __device__ Load load(int w, const StageInfo &si) const { return grad_load(si, w < t.n_items); }
    __device__ void consume(int w, uint8_t *stage, const StageInfo &si, uint32_t *scratch, int warp, int lane) const
    {
        if (w < t.n_items)
            absmax_chunk(si, reinterpret_cast<const float4 *>(stage), amax, warp, lane);
        else
            quant_chunk<C, true>(t, c, si, stage, stage + kF32Bytes, scratch, avg, warp, lane);
    }
    __device__ void after_phase_a_last(int) const {}
};

// ------------------------------------------------------------------ the engine
template <class Op>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const Op op, uint32_t *done_ctr, uint32_t target)
{
    using Cfg = StageCfg<Op::kCodeBytes>;
    using Smem = StreamSmem<Cfg::kStages, Cfg::kStageBytes>;
    constexpr int NS = Cfg::kStages;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&S.full[s], 2);  // load arrival + "side info final" arrival
            mbar_init(&S.empty[s], kConsWarps);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    const int nw = op.n_work();
    const int G = gridDim.x;
    const int my_items = nw > (int)blockIdx.x ? (nw - 1 - (int)blockIdx.x) / G + 1 : 0;
    const int na = op.n_phase_a();
    const int my_a = na > (int)blockIdx.x ? (na - 1 - (int)blockIdx.x) / G + 1 : 0;  // my phase-A items (first)

    if (warp == kConsWarps) {  // ---------------- producer warp
        const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
        bool ready = !op.waits();
        int pend_lo = 0, pend_hi = 0;  // my items [pend_lo, pend_hi) issued, f~ still owed
        // finalize: wait for the abs-max pass, then supply f~ to the owed stages
        // and to the not-yet-issued entries of the current batch.
        auto finalize = [&](int b0, int n_in) {
            if (!ready) {
                if (lane == 0)
                    spin_until([&] { return (int)(ld_acquire(done_ctr) - target) >= 0; }, op.t.flag);
                __syncwarp();
                ready = true;
                for (int i = pend_lo + lane; i < pend_hi; i += 32) {
                    StageInfo &si = S.info[i % NS];
                    si.ft = op.late_ft(si);
                    si.ft_ok = 1;
                }
                for (int j = lane; j < n_in; j += 32)
                    if (b0 + j >= pend_hi && !S.batch[j].ft_ok) {
                        S.batch[j].ft = op.late_ft(S.batch[j]);
                        S.batch[j].ft_ok = 1;
                    }
                __syncwarp();
            }
            if (lane == 0)
                for (int i = pend_lo; i < pend_hi; ++i) mbar_arrive(&S.full[i % NS]);
            pend_lo = pend_hi;
        };
        StageInfo next;
        if (lane < my_items) next = op.fetch(blockIdx.x + lane * G, ready);
        for (int b0 = 0; b0 < my_items; b0 += 32) {
            if (ready && lane < my_items - b0 && !next.ft_ok) {  // fetched before the abs-max pass ended
                next.ft = op.late_ft(next);
                next.ft_ok = 1;
            }
            __syncwarp();
            S.batch[lane] = next;
            __syncwarp();
            const int n_in = min(32, my_items - b0);
            if (b0 + 32 + lane < my_items) next = op.fetch(blockIdx.x + (b0 + 32 + lane) * G, ready);
            for (int j = 0; j < n_in; ++j) {
                const int i = b0 + j;
                const int s = i % NS;
                // the stage's previous occupant may still owe its f~: supply it first
                if (pend_lo < pend_hi && pend_lo <= i - NS) finalize(b0, n_in);
                if (lane == 0) {
                    mbar_wait(&S.empty[s], ((uint32_t)(i / NS) & 1u) ^ 1u);
                    const StageInfo si = S.batch[j];
                    S.info[s] = si;
                    const Load ld = op.load(blockIdx.x + i * G, si);
                    mbar_arrive_expect_tx(&S.full[s], ld.bytes);
                    if (ld.bytes)
                        bulk_g2s(S.stage[s] + ld.dst_off, ld.src, ld.bytes, &S.full[s], ld.keep ? keep : stream);
                }
                __syncwarp();
                if (!S.batch[j].ft_ok) {
                    ++pend_hi;  // f~ owed: the second arrival comes from finalize
                    int done = 0;
                    if (lane == 0) done = (int)(ld_acquire(done_ctr) - target) >= 0;
                    if (__shfl_sync(0xffffffffu, done, 0)) finalize(b0, n_in);
                } else {
                    if (pend_lo < pend_hi) finalize(b0, n_in);  // keep arrivals in order
                    if (lane == 0) mbar_arrive(&S.full[s]);
                    pend_lo = pend_hi = i + 1;
                }
            }
        }
        if (pend_lo < pend_hi) finalize(my_items, 0);
        return;
    }

    // ---------------- consumers
    // end of my abs-max pass: make my red.max visible, count the CTA done
    // (a CTA with no abs-max item counts itself done before anything else:
    // its quantise items wait for the count)
    auto count_done = [&]() {
        if (lane == 0) __threadfence();
        bar_consumers();
        if (threadIdx.x == 0) S.flag = (int)(atom_add_acq_rel(done_ctr, 1u) == target - 1u);
        bar_consumers();
        if (S.flag) op.after_phase_a_last(threadIdx.x);
    };
    if (na > 0 && my_a == 0) count_done();
    for (int i = 0; i < my_items; ++i) {
        const int s = i % NS;
        mbar_wait(&S.full[s], (uint32_t)(i / NS) & 1u);
        op.consume(blockIdx.x + i * G, S.stage[s], S.info[s], S.scratch[warp], warp, lane);
        if (lane == 0) {
            bulk_commit();
            bulk_wait_read();  // the stage may be refilled once the bulk stores have read it
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        if (i == my_a - 1) count_done();
    }
    if (lane == 0) bulk_wait_all();
}

// ------------------------------------------------------------------ launch
int stream_grid(int n_work) { return std::max(1, std::min(n_work, sm_count())); }

template <class Op>
static cudaError_t launch_stream(const Op &op, int n_work, bool cooperative, uint32_t *done_ctr, uint32_t target,
                                 cudaStream_t s)
{
    using Cfg = StageCfg<Op::kCodeBytes>;
    using Smem = StreamSmem<Cfg::kStages, Cfg::kStageBytes>;
    static bool configured = false;
    const size_t smem = sizeof(Smem) + 1024;  // + alignment slack
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(stream_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (n_work <= 0) return cudaSuccess;
    const int grid = stream_grid(n_work);  // one CTA per SM (the stages take most of shared memory)
    if (cooperative) {
        void *args[] = {const_cast<Op *>(&op), &done_ctr, &target};
        return cudaLaunchCooperativeKernel((const void *)stream_kernel<Op>, dim3(grid), dim3(kStreamThreads), args,
                                           smem, s);
    }
    stream_kernel<Op><<<grid, kStreamThreads, smem, s>>>(op, done_ctr, target);
    return cudaGetLastError();
}

cudaError_t launch_stream_absmax(const DevTables &t, int world, uint32_t gen, uint32_t target, cudaStream_t s)
{
    uint32_t *cur = t.amax2 + (size_t)(gen & 1u) * t.n_layers, *other = t.amax2 + (size_t)((gen + 1u) & 1u) * t.n_layers;
    return launch_stream(AbsmaxOp{t, cur, other, target, world}, t.n_items, false, t.done, target, s);
}

cudaError_t launch_stream_quant(const DevTables &t, int e, int m, bool hw, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        if constexpr (C::kB == 0) {
            return cudaErrorNotSupported;  // runtime formats use the simple kernels
        } else {
            return launch_stream(QuantOp<C>{t, c, bias}, t.n_items, false, t.done, 0u, s);
        }
    });
}

cudaError_t launch_stream_unpack(const DevTables &t, int e, int m, bool hw, int world, int average, cudaStream_t s)
{
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        if constexpr (C::kB == 0) {
            return cudaErrorNotSupported;
        } else {
            return launch_stream(UnpackOp<C>{t, c, world, average}, t.n_items, false, t.done, 0u, s);
        }
    });
}

bool stream_fused_supported(int e, int m, bool hw)
{
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
               using C = decltype(c);
               return C::kB == 0 ? cudaErrorNotSupported : cudaSuccess;
           }) == cudaSuccess;
}

cudaError_t launch_stream_fused_p1(const DevTables &t, int e, int m, bool hw, int average, uint32_t gen,
                                   uint32_t target, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    uint32_t *cur = t.amax2 + (size_t)(gen & 1u) * t.n_layers, *other = t.amax2 + (size_t)((gen + 1u) & 1u) * t.n_layers;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        if constexpr (C::kB == 0) {
            return cudaErrorNotSupported;
        } else {
            return launch_stream(FusedP1Op<C>{t, c, cur, other, target, bias, average}, 2 * t.n_items, true, t.done,
                                 target, s);
        }
    });
}

}  // namespace aps
