// aps_stream.cu -- persistent, TMA-bulk pipelined versions of the HBM-bound
// APS kernels for sm_100a.
//
// Every hot kernel of the path streams each gradient element through the SM
// once per pass (4 B read, b/8 B written, or the reverse), so it is bound by
// HBM bandwidth, and short (~20 us at ResNet-50 size): CTA launch ramp and
// tail matter as much as steady-state bandwidth.  The engine therefore runs
// ONE persistent CTA per SM:
//   warp 8 (producer, one elected lane): for each work item assigned to the
//     CTA (static round-robin), waits for a free stage, arms the stage's
//     mbarrier with the byte count and issues one cp.async.bulk
//     global->shared copy (the TMA bulk-copy engine; up to 32 KB per item),
//     with an L2 eviction-priority hint;
//   warps 0..7 (consumers): wait on the stage's mbarrier, compute from shared
//     memory, write results with coalesced 128-bit stores, and release the
//     stage.
// Six 32 KB stages give 192 KB in flight per SM (~28 MB chip-wide), far
// above the bandwidth-latency product, with no registers tied up in loads.
//
// Fused p = 1 path (launch_stream_fused_p1): with one rank there is no
// collective between FindMaxExp and Cast, so a single launch does
//   phase A  abs-max of every work item (forward order; L2 evict_last hint),
//            the last item of a layer publishes E_l with a release store of
//            the call's generation stamp;
//   phase B  per item, in REVERSE order: wait (acquire) for E_l, then
//            f~, scale, Cast, pack (codes to the packed buffer) and
//            Cast back, unscale, average -> fp32 output.
// Reverse order makes the second read of the gradients hit the data phase A
// left in the 126 MB L2 most recently.  Every CTA finishes all of its phase A
// items before its first phase B item and the grid is co-resident
// (cooperative launch), so the waits cannot deadlock.
#include <cstdint>
#include <algorithm>
#include <climits>

#include "aps_device.cuh"

namespace aps {

constexpr int kStageBytes = kItemTiles * kTile * 4;  // 32 KB: one work item of fp32
constexpr int kStages = 6;
constexpr int kConsWarps = 8;
constexpr int kConsThreads = kConsWarps * 32;
constexpr int kStreamThreads = kConsThreads + 32;

struct StreamSmem {
    alignas(128) uint8_t stage[kStages][kStageBytes];
    alignas(8) uint64_t full[kStages];
    uint64_t empty[kStages];
    uint32_t red[2][kConsWarps];
    int32_t bcast[2];
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
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bar_consumers()
{
    asm volatile("bar.sync 1, %0;" ::"n"(kConsThreads) : "memory");
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
    uint32_t bytes;  // multiple of 16
    bool keep;       // L2 evict_last (data will be read again) vs evict_first
};

// ------------------------------------------------------------------ the engine
template <class Op>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const Op op)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    StreamSmem &S = *reinterpret_cast<StreamSmem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kConsWarps);
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    const int nw = op.n_work();
    if (warp == kConsWarps) {  // ---------------- producer
        if (lane == 0) {
            const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
            int i = 0;
            for (int w = blockIdx.x; w < nw; w += gridDim.x, ++i) {
                const int s = i % kStages;
                const uint32_t ph = (uint32_t)(i / kStages) & 1u;
                mbar_wait(&S.empty[s], ph ^ 1u);
                const Load ld = op.load(w);
                mbar_arrive_expect_tx(&S.full[s], ld.bytes);
                if (ld.bytes) bulk_g2s(S.stage[s], ld.src, ld.bytes, &S.full[s], ld.keep ? keep : stream);
            }
        }
        return;
    }
    // ---------------- consumers
    int i = 0;
    for (int w = blockIdx.x; w < nw; w += gridDim.x, ++i) {
        const int s = i % kStages;
        const uint32_t ph = (uint32_t)(i / kStages) & 1u;
        mbar_wait(&S.full[s], ph);
        op.process(w, S.stage[s], S, i);
        if (Op::kWritesStage) fence_proxy_async_smem();  // generic writes before the next TMA write
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
    }
}

// ------------------------------------------------------------------ item helpers
struct ItemView {
    Item it;
    LayerDev L;
    int64_t begin;  // first element of the item within the layer
    int cnt;        // valid elements in the item
};

__device__ __forceinline__ ItemView view(const DevTables &t, int k)
{
    ItemView v;
    v.it = t.items[k];
    v.L = t.layers[v.it.layer];
    v.begin = (int64_t)v.it.tile_begin * kTile;
    v.cnt = (int)min((int64_t)v.it.n_tiles * kTile, v.L.numel - v.begin);
    return v;
}

__device__ __forceinline__ Load grad_load(const DevTables &t, int k, bool keep)
{
    const ItemView v = view(t, k);
    return Load{t.src[v.it.layer] + v.begin, (uint32_t)(v.cnt >> 2) * 16u, keep};
}

// fp32 group j (elements 4j..4j+3) of an item: from the stage when it was
// bulk-copied, else (the < 4-element tail of a layer) from global memory.
__device__ __forceinline__ float4 stage_group(const uint8_t *stage, const float *g, int j, int cnt)
{
    if (4 * j + 4 <= cnt) return reinterpret_cast<const float4 *>(stage)[j];
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int e0 = 4 * j;
    if (e0 + 0 < cnt) v.x = g[e0 + 0];
    if (e0 + 1 < cnt) v.y = g[e0 + 1];
    if (e0 + 2 < cnt) v.z = g[e0 + 2];
    return v;
}

// a1: abs-max of the item, combined per layer; the last item of a layer
// writes E_l (and, when gen != 0, publishes it with a release store).
__device__ __forceinline__ void absmax_consume(const DevTables &t, int N, const ItemView &v, const uint8_t *stage,
                                               StreamSmem &S, int i, uint32_t gen)
{
    const int n4 = v.cnt >> 2;
    const float4 *s4 = reinterpret_cast<const float4 *>(stage);
    uint32_t mx = 0;
#pragma unroll 8
    for (int j = threadIdx.x; j < n4; j += kConsThreads) mx = max(mx, absbits4(s4[j]));
    if ((int)threadIdx.x < (v.cnt & 3))
        mx = max(mx, __float_as_uint(t.src[v.it.layer][v.begin + 4 * n4 + threadIdx.x]) & 0x7fffffffu);
    mx = __reduce_max_sync(0xffffffffu, mx);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) S.red[i & 1][warp] = mx;
    bar_consumers();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < kConsWarps; ++k) m = max(m, S.red[i & 1][k]);
        const int l = v.it.layer;
        atomicMax(&t.amax[l], m);
        __threadfence();
        const uint32_t done = atomicAdd(&t.count[l], 1u);
        if (done == (uint32_t)v.L.n_items - 1u) {
            __threadfence();
            const uint32_t A = atomicExch(&t.amax[l], 0u);
            t.count[l] = 0u;
            t.E_local[l] = exponent_of(A, N);
            if (gen) {
                __threadfence();
                st_release(&t.ready[l], gen);
            }
        }
    }
}

// a3+a4 (+ a7 when Fuse): scale, Cast, pack; optionally Cast back, unscale
template <int B, class C, bool Fuse>
__device__ __forceinline__ void quant_consume_direct(const DevTables &t, const C &c, const ItemView &v,
                                                     const uint8_t *stage, int ft, int N, int avg)
{
    using W = typename Word4<B>::T;
    W *out = reinterpret_cast<W *>(t.packed + (v.L.tile_off + v.it.tile_begin) * (16 * B));
    const float *g = t.src[v.it.layer] + v.begin;
    float *o = Fuse ? t.dst[v.it.layer] + v.begin : nullptr;
    const Pow2 s(ft);
    const Unscale us(ft, N, avg);
    const int ng = v.it.n_tiles * (kTile / 4);
    if (!s.wide) {
#pragma unroll 4
        for (int j = threadIdx.x; j < ng; j += kConsThreads) {
            const float4 x = stage_group(stage, g, j, v.cnt);
            const float4 y = make_float4(__fmul_rn(x.x, s.f), __fmul_rn(x.y, s.f), __fmul_rn(x.z, s.f),
                                         __fmul_rn(x.w, s.f));
            const W code = pack4<B>(c, y);
            out[j] = code;
            if (Fuse) store_group(o, 4 * j, v.cnt, us.apply4(unpack4<B>(c, code)));
        }
    } else {
        for (int j = threadIdx.x; j < ng; j += kConsThreads) {
            const W code = pack4<B>(c, s.apply4(stage_group(stage, g, j, v.cnt)));
            out[j] = code;
            if (Fuse) store_group(o, 4 * j, v.cnt, us.apply4(unpack4<B>(c, code)));
        }
    }
}

template <class C, bool Fuse>
__device__ __forceinline__ void quant_consume_tile(const DevTables &t, const C &c, const ItemView &v,
                                                   uint8_t *stage, int ft, int N, int avg)
{
    const int b = c.b();
    uint32_t *out = reinterpret_cast<uint32_t *>(t.packed) + (v.L.tile_off + v.it.tile_begin) * (4 * b);
    const float *g = t.src[v.it.layer] + v.begin;
    float *o = Fuse ? t.dst[v.it.layer] + v.begin : nullptr;
    const Pow2 s(ft);
    const Unscale us(ft, N, avg);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *codes_all = reinterpret_cast<uint32_t *>(stage);
    for (int tt = warp; tt < v.it.n_tiles; tt += kConsWarps) {
        const int j = tt * (kTile / 4) + lane;
        const float4 y = s.apply4(stage_group(stage, g, j, v.cnt));
        const uint4 cd = make_uint4(c.enc(y.x), c.enc(y.y), c.enc(y.z), c.enc(y.w));
        uint32_t *codes = codes_all + tt * kTile;  // in place over the tile's fp32
        __syncwarp();
        *reinterpret_cast<uint4 *>(codes + 4 * lane) = cd;
        __syncwarp();
        uint32_t *ow = out + (int64_t)tt * (4 * b);
        for (int w = lane; w < 4 * b; w += 32) ow[w] = assemble_word(codes, w, b);
        if (Fuse) {
            const float4 d = make_float4(c.dec(cd.x), c.dec(cd.y), c.dec(cd.z), c.dec(cd.w));
            store_group(o, 4 * j, v.cnt, us.apply4(d));
        }
    }
}

// ------------------------------------------------------------------ ops
struct AbsmaxOp {
    static constexpr bool kWritesStage = false;
    DevTables t;
    int N;
    __device__ int n_work() const { return t.n_items; }
    __device__ Load load(int w) const { return grad_load(t, w, true); }
    __device__ void process(int w, uint8_t *stage, StreamSmem &S, int i) const
    {
        absmax_consume(t, N, view(t, w), stage, S, i, 0u);
    }
};

// f~ of a layer (Alg. 1 line 4) from the final E, broadcast to the consumers
__device__ __forceinline__ int layer_ftilde(const DevTables &t, const ItemView &v, int bias, StreamSmem &S, int i,
                                            uint32_t gen)
{
    if (threadIdx.x == 0) {
        if (gen)
            while (ld_acquire(&t.ready[v.it.layer]) != gen) __nanosleep(32);
        S.bcast[i & 1] = scale_exponent(t, v.it.layer, bias, v.it.tile_begin == 0);
    }
    bar_consumers();
    return S.bcast[i & 1];
}

template <class C>
struct QuantOp {
    static constexpr bool kWritesStage = !(C::kB == 8 || C::kB == 16 || C::kB == 32);
    DevTables t;
    C c;
    int bias;
    // reverse order: the items phase a1 read last are still in L2
    __device__ int n_work() const { return t.n_items; }
    __device__ int item(int w) const { return t.n_items - 1 - w; }
    __device__ Load load(int w) const { return grad_load(t, item(w), false); }
    __device__ void process(int w, uint8_t *stage, StreamSmem &S, int i) const
    {
        const ItemView v = view(t, item(w));
        const int ft = layer_ftilde(t, v, bias, S, i, 0u);
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32)
            quant_consume_direct<C::kB, C, false>(t, c, v, stage, ft, 1, 0);
        else
            quant_consume_tile<C, false>(t, c, v, stage, ft, 1, 0);
    }
};

template <class C>
struct UnpackOp {
    static constexpr bool kWritesStage = false;
    DevTables t;
    C c;
    int N, avg;
    __device__ int n_work() const { return t.n_items; }
    __device__ Load load(int w) const
    {
        const Item it = t.items[w];
        const LayerDev L = t.layers[it.layer];
        const int b = c.b();
        return Load{t.packed + (L.tile_off + it.tile_begin) * (16 * b), (uint32_t)(16 * b * it.n_tiles), false};
    }
    __device__ void process(int w, uint8_t *stage, StreamSmem &S, int i) const
    {
        const ItemView v = view(t, w);
        const Unscale us(t.ftilde[v.it.layer], N, avg);
        float *o = t.dst[v.it.layer] + v.begin;
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32) {
            using W = typename Word4<C::kB>::T;
            const W *in = reinterpret_cast<const W *>(stage);
            const int ng = (v.cnt + 3) >> 2;
#pragma unroll 4
            for (int j = threadIdx.x; j < ng; j += kConsThreads)
                store_group(o, 4 * j, v.cnt, us.apply4(unpack4<C::kB>(c, in[j])));
        } else {
            const int b = c.b();
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            const uint32_t *words_all = reinterpret_cast<const uint32_t *>(stage);
            for (int tt = warp; tt < v.it.n_tiles; tt += kConsWarps) {
                const uint32_t *words = words_all + tt * (4 * b);  // words[4b] reads the next tile / pad: masked
                const int k0 = lane * 4;
                const float4 d = make_float4(c.dec(extract_code(words, k0, b)), c.dec(extract_code(words, k0 + 1, b)),
                                             c.dec(extract_code(words, k0 + 2, b)),
                                             c.dec(extract_code(words, k0 + 3, b)));
                store_group(o, tt * kTile + k0, v.cnt, us.apply4(d));
            }
        }
    }
};

template <class C>
struct FusedP1Op {
    static constexpr bool kWritesStage = !(C::kB == 8 || C::kB == 16 || C::kB == 32);
    DevTables t;
    C c;
    int bias, avg;
    uint32_t gen;
    __device__ int n_work() const { return 2 * t.n_items; }
    __device__ Load load(int w) const
    {
        return w < t.n_items ? grad_load(t, w, true) : grad_load(t, 2 * t.n_items - 1 - w, false);
    }
    __device__ void process(int w, uint8_t *stage, StreamSmem &S, int i) const
    {
        if (w < t.n_items) {
            absmax_consume(t, 1, view(t, w), stage, S, i, gen);
            return;
        }
        const ItemView v = view(t, 2 * t.n_items - 1 - w);
        const int ft = layer_ftilde(t, v, bias, S, i, gen);
        if constexpr (C::kB == 8 || C::kB == 16 || C::kB == 32)
            quant_consume_direct<C::kB, C, true>(t, c, v, stage, ft, 1, avg);
        else
            quant_consume_tile<C, true>(t, c, v, stage, ft, 1, avg);
    }
};

// ------------------------------------------------------------------ launch
template <class Op>
static cudaError_t launch_stream(const Op &op, int n_work, bool cooperative, cudaStream_t s)
{
    static bool configured = false;
    static int blocks_per_sm = 1;
    const size_t smem = sizeof(StreamSmem);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(stream_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, stream_kernel<Op>, kStreamThreads, smem);
        if (e != cudaSuccess) return e;
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
        configured = true;
    }
    if (n_work <= 0) return cudaSuccess;
    const int grid = std::min(n_work, sm_count() * blocks_per_sm);
    if (cooperative) {
        void *args[] = {const_cast<Op *>(&op)};
        return cudaLaunchCooperativeKernel((const void *)stream_kernel<Op>, dim3(grid), dim3(kStreamThreads), args,
                                           smem, s);
    }
    stream_kernel<Op><<<grid, kStreamThreads, smem, s>>>(op);
    return cudaGetLastError();
}

cudaError_t launch_stream_absmax(const DevTables &t, int world, cudaStream_t s)
{
    return launch_stream(AbsmaxOp{t, world}, t.n_items, false, s);
}

cudaError_t launch_stream_quant(const DevTables &t, int e, int m, bool hw, cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        if constexpr (C::kB == 0) {
            return cudaErrorNotSupported;  // runtime formats use the simple kernels
        } else {
            return launch_stream(QuantOp<C>{t, c, bias}, t.n_items, false, s);
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
            return launch_stream(UnpackOp<C>{t, c, world, average}, t.n_items, false, s);
        }
    });
}

cudaError_t launch_stream_fused_p1(const DevTables &t, int e, int m, bool hw, int average, uint32_t gen,
                                   cudaStream_t s)
{
    const int bias = (1 << (e - 1)) - 1;
    return with_codec(e, m, hw, [&](auto c) -> cudaError_t {
        using C = decltype(c);
        if constexpr (C::kB == 0) {
            return cudaErrorNotSupported;
        } else {
            return launch_stream(FusedP1Op<C>{t, c, bias, average, gen}, 2 * t.n_items, true, s);
        }
    });
}

}  // namespace aps
