// microbench_stream.cu -- B200 streaming-bandwidth microbenchmarks that
// decide the design of libaps's HBM-bound kernels:
//   ldg   : grid of many CTAs, 128-bit ld.global.nc.L1::no_allocate, K loads in flight per thread
//   tma   : persistent 1 CTA/SM, producer lane issuing cp.async.bulk of R bytes into S stages,
//           consumers reduce from shared memory (abs-max), L2 policy none/first/last
//   stg   : grid of many CTAs, 128-bit st.global
//   tmast : persistent, bulk shared->global stores of R bytes
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb microbench_stream.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(uint64_t *b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) { while (!mbar_try(b, ph)) {} }

__global__ void k_ldg(const float4 *__restrict__ in, size_t n4, uint32_t *out)
{
    uint32_t mx = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x * 8 + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
    for (; i < n4; i += stride) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            size_t j = i + (size_t)k * blockDim.x;
            if (j < n4) asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(in + j));
            else v[k] = make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) mx = max(mx, max(max(__float_as_uint(v[k].x), __float_as_uint(v[k].y)), max(__float_as_uint(v[k].z), __float_as_uint(v[k].w))) & 0x7fffffffu);
    }
    mx = __reduce_max_sync(~0u, mx);
    if ((threadIdx.x & 31) == 0 && mx == 0x12345678u) out[0] = mx;
}

__global__ void k_stg(float4 *out, size_t n4)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n4; i += (size_t)gridDim.x * blockDim.x) out[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}

template <int POL>
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol)
{
    if (POL == 0)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
    else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// persistent TMA-load stream: item = R bytes; S stages; 8 consumer warps + 1 producer warp
template <int POL>
__global__ void __launch_bounds__(288, 1) k_tma(const uint8_t *in, size_t nbytes, int R, int S, uint32_t *out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)S * R);
    uint64_t *empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t nitems = nbytes / R;
    if (warp == 8) {
        if (lane == 0) {
            uint64_t pol;
            if (POL == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            int i = 0;
            for (size_t w = blockIdx.x; w < nitems; w += gridDim.x, ++i) {
                int s = i % S; uint32_t ph = (i / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect(&full[s], R);
                bulk_load<POL>(sm + (size_t)s * R, in + w * R, R, &full[s], pol);
            }
        }
        return;
    }
    uint32_t mx = 0;
    int i = 0;
    for (size_t w = blockIdx.x; w < nitems; w += gridDim.x, ++i) {
        int s = i % S; uint32_t ph = (i / S) & 1;
        mbar_wait(&full[s], ph);
        const float4 *s4 = reinterpret_cast<const float4 *>(sm + (size_t)s * R);
        for (int j = threadIdx.x; j < R / 16; j += 256) {
            float4 v = s4[j];
            mx = max(mx, max(max(__float_as_uint(v.x), __float_as_uint(v.y)), max(__float_as_uint(v.z), __float_as_uint(v.w))) & 0x7fffffffu);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (mx == 0x12345678u) out[0] = mx;
}

// persistent TMA-store stream: consumers fill a stage, lane 0 of each warp bulk-stores its slice
__global__ void __launch_bounds__(256, 1) k_tmast(uint8_t *outp, size_t nbytes, int R, int S)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nitems = nbytes / R;
    const int slice = R / 8;
    int i = 0;
    for (size_t w = blockIdx.x; w < nitems; w += gridDim.x, ++i) {
        int s = i % S;
        float4 *s4 = reinterpret_cast<float4 *>(sm + (size_t)s * R + warp * slice);
        if (lane == 0 && i >= S) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
        __syncwarp();
        for (int j = lane; j < slice / 16; j += 32) s4[j] = make_float4(1.f, 2.f, 3.f, (float)j);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(outp + w * R + warp * slice), "r"(smem_u32(s4)), "r"(slice) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// persistent LDG stream: grid = SMs * k, each thread keeps 8 float4 in flight, items of R bytes
__global__ void k_ldg_items(const uint8_t *in, size_t nbytes, int R, uint32_t *out)
{
    const size_t nitems = nbytes / R;
    uint32_t mx = 0;
    for (size_t w = blockIdx.x; w < nitems; w += gridDim.x) {
        const float4 *p = reinterpret_cast<const float4 *>(in + w * R);
        for (int base = 0; base < R / 16; base += 8 * blockDim.x) {
            float4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                int j = base + threadIdx.x + k * blockDim.x;
                if (j < R / 16) asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(p + j));
                else v[k] = make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) mx = max(mx, max(max(__float_as_uint(v[k].x), __float_as_uint(v[k].y)), max(__float_as_uint(v[k].z), __float_as_uint(v[k].w))) & 0x7fffffffu);
        }
    }
    mx = __reduce_max_sync(~0u, mx);
    if ((threadIdx.x & 31) == 0 && mx == 0x12345678u) out[0] = mx;
}

int main(int argc, char **argv)
{
    const size_t nbytes = argc > 1 ? (size_t)atoll(argv[1]) : (size_t)1 << 30;
    const bool quick = argc > 2;
    printf("=== %zu bytes per pass\n", nbytes);
    uint8_t *a, *b;
    uint32_t *o;
    CK(cudaMalloc(&a, nbytes));
    CK(cudaMalloc(&b, nbytes));
    CK(cudaMalloc(&o, 64));
    CK(cudaMemset(a, 0x3c, nbytes));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, const char *name, double bytes) {
        for (int w = 0; w < 2; ++w) launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        printf("%-44s %8.1f GB/s  (%.3f ms)\n", name, bytes / (best * 1e-3) / 1e9, best);
    };
    char nm[128];
    for (int ctas : {sms, 2 * sms, 4 * sms, 8 * sms, 32 * sms}) {
        snprintf(nm, sizeof nm, "ldg v4x8 grid=%d x256", ctas);
        timeit([&] { k_ldg<<<ctas, 256>>>((const float4 *)a, nbytes / 16, o); }, nm, (double)nbytes);
    }
    for (int k : {1, 2, 4, 8}) {
        for (int R : {8192, 32768}) {
            snprintf(nm, sizeof nm, "ldg persistent items R=%dK grid=%dxSM x256", R / 1024, k);
            timeit([&] { k_ldg_items<<<k * sms, 256>>>(a, nbytes, R, o); }, nm, (double)nbytes);
        }
    }
    for (int ctas : {sms, 4 * sms, 16 * sms}) {
        snprintf(nm, sizeof nm, "stg v4 grid=%d x256", ctas);
        timeit([&] { k_stg<<<ctas, 256>>>((float4 *)b, nbytes / 16); }, nm, (double)nbytes);
    }
    for (int pol = 0; pol < (quick ? 1 : 3); ++pol) {
        for (int R : {4096, 8192, 16384, 32768}) {
            for (int S : {2, 4, 6, 12, 24, 48}) {
                if (quick && !(S == 4 || S == 6)) continue;
                size_t smem = (size_t)S * R + 2 * S * 8 + 64;
                if (smem > 220 * 1024) continue;
                auto kern = pol == 0 ? k_tma<0> : pol == 1 ? k_tma<1> : k_tma<2>;
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                snprintf(nm, sizeof nm, "tma-load pol=%s R=%dK S=%d", pol == 0 ? "none" : pol == 1 ? "first" : "last", R / 1024, S);
                timeit([&] { kern<<<sms, 288, smem>>>(a, nbytes, R, S, o); }, nm, (double)nbytes);
            }
        }
    }
    for (int R : {8192, 32768}) {
        for (int S : {2, 4, 6}) {
            size_t smem = (size_t)S * R;
            if (smem > 220 * 1024) continue;
            CK(cudaFuncSetAttribute(k_tmast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            snprintf(nm, sizeof nm, "tma-store R=%dK S=%d", R / 1024, S);
            timeit([&] { k_tmast<<<sms, 256, smem>>>(b, nbytes, R, S); }, nm, (double)nbytes);
        }
    }
    return 0;
}
