// microbench_fused.cu -- what schedule can move the N = 1 APS sync's bytes at HBM speed?
// One "step" = the ResNet-50-sized traffic of the fused sync: read g (L fp32), write
// codes (L bytes) and out (L fp32).  Steady state: K steps back to back, rotating over S
// buffer sets (> L2), one event pair.  Kernels (no APS dependency logic, just the bytes
// and a representative amount of ALU: scale, cvt e5m2x2, cvt back, unscale):
//   max   : read-only abs-max pass (grid-stride LDG)
//   qu    : quantise+unscale pass, grid-stride LDG, 8 float4 in flight per thread
//   qu_tma: quantise+unscale pass, persistent, producer warp bulk-loads 32 KB stages
//   pair  : max then qu (reverse order) -- the two-kernel schedule
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mbf microbench_fused.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

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

__device__ __forceinline__ float4 ldnc(const float4 *p, uint64_t pol, bool hint)
{
    float4 r;
    if (hint)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t absbits4(float4 v)
{
    return max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
               max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu));
}
__device__ __forceinline__ uint32_t enc2(float hi, float lo)
{
    uint16_t d;
    asm("cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2;" : "=h"(d) : "f"(hi), "f"(lo));
    return d;
}
__device__ __forceinline__ float2 dec2(uint32_t two)
{
    uint32_t h2;
    asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)two));
    return __half22float2(*reinterpret_cast<__half2 *>(&h2));
}
// quantise 4 values -> packed word and unscaled outputs
__device__ __forceinline__ void qu4(float4 v, float s, float is, uint32_t &code, float4 &o)
{
    const uint32_t lo = enc2(v.y * s, v.x * s), hi = enc2(v.w * s, v.z * s);
    code = lo | (hi << 16);
    const float2 a = dec2(lo), b = dec2(hi);
    o = make_float4(a.x * is, a.y * is, b.x * is, b.y * is);
}

__global__ void __launch_bounds__(256) k_max(const float4 *__restrict__ in, size_t n4, uint32_t *out, int hint)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    uint32_t mx = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
    for (size_t i = blockIdx.x * (size_t)blockDim.x * 8 + threadIdx.x; i < n4; i += stride) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const size_t j = i + (size_t)k * blockDim.x;
            v[k] = j < n4 ? ldnc(in + j, pol, hint) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) mx = max(mx, absbits4(v[k]));
    }
    mx = __reduce_max_sync(~0u, mx);
    if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// grid-stride quantise pass; rev = walk the blocks in reverse (L2 reuse after k_max)
__global__ void __launch_bounds__(256) k_qu(const float4 *__restrict__ in, uint32_t *__restrict__ codes,
                                           float4 *__restrict__ out, size_t n4, int rev, int sthint)
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const size_t per = (size_t)blockDim.x * 8;
    const size_t nblk = (n4 + per - 1) / per;
    for (size_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        const size_t bb = rev ? nblk - 1 - b : b;
        const size_t i = bb * per + threadIdx.x;
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const size_t j = i + (size_t)k * blockDim.x;
            v[k] = j < n4 ? ldnc(in + j, pol, true) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const size_t j = i + (size_t)k * blockDim.x;
            uint32_t c;
            float4 o;
            qu4(v[k], 1024.f, 1.f / 1024.f, c, o);
            if (j < n4) {
                if (sthint) {
                    asm volatile("st.global.L1::no_allocate.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(codes + j), "r"(c), "l"(pol) : "memory");
                    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(out + j), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w), "l"(pol) : "memory");
                } else {
                    codes[j] = c;
                    out[j] = o;
                }
            }
        }
    }
}

// persistent TMA-fed quantise pass: 1 producer warp + 8 consumer warps, S stages of R bytes
__global__ void __launch_bounds__(288, 1) k_qu_tma(const uint8_t *in, uint32_t *codes, float4 *out, size_t nbytes,
                                                   int R, int S, int rev)
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
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int i = 0;
            for (size_t w = blockIdx.x; w < nitems; w += gridDim.x, ++i) {
                const size_t ww = rev ? nitems - 1 - w : w;
                int s = i % S; uint32_t ph = (i / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect(&full[s], R);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                             ::"r"(smem_u32(sm + (size_t)s * R)), "l"(in + ww * R), "r"(R), "r"(smem_u32(&full[s])), "l"(pol) : "memory");
            }
        }
        return;
    }
    int i = 0;
    for (size_t w = blockIdx.x; w < nitems; w += gridDim.x, ++i) {
        const size_t ww = rev ? nitems - 1 - w : w;
        int s = i % S; uint32_t ph = (i / S) & 1;
        mbar_wait(&full[s], ph);
        const float4 *s4 = reinterpret_cast<const float4 *>(sm + (size_t)s * R);
        const size_t base = ww * (R / 16);
        float4 v[8];
        const int per = R / 16 / 256;  // float4 per thread
        for (int k0 = 0; k0 < per; k0 += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = s4[threadIdx.x + (k0 + k) * 256];
            if (k0 + 8 >= per) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t c;
                float4 o;
                qu4(v[k], 1024.f, 1.f / 1024.f, c, o);
                const size_t j = base + threadIdx.x + (k0 + k) * 256;
                codes[j] = c;
                out[j] = o;
            }
        }
    }
}

int main(int argc, char **argv)
{
    const size_t L = argc > 1 ? (size_t)atoll(argv[1]) : 25557032 / 8192 * 8192;  // ResNet-50 elements (8192-multiple)
    const int S = argc > 2 ? atoi(argv[2]) : 3;   // rotating buffer sets
    const int K = 60;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<float *> g(S), o(S);
    std::vector<uint32_t *> c(S);
    for (int s = 0; s < S; ++s) {
        CK(cudaMalloc(&g[s], 4 * L));
        CK(cudaMalloc(&o[s], 4 * L));
        CK(cudaMalloc(&c[s], L));
        CK(cudaMemset(g[s], 0x3c, 4 * L));
    }
    uint32_t *mx;
    CK(cudaMalloc(&mx, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double step_bytes = 4.0 * L + 1.0 * L + 4.0 * L;
    printf("=== L = %zu elements, %d rotating sets, %d steps; DRAM floor per step %.1f MB\n", L, S, K, step_bytes / 1e6);
    auto timeit = [&](const char *name, double bytes, auto step) {
        for (int k = 0; k < 2 * S; ++k) step(k);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int k = 0; k < K; ++k) step(k);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = ms * 1e3 / K;
        printf("%-52s %8.2f us/step  %7.1f GB/s (of %.0f MB)\n", name, us, bytes / (us * 1e-6) / 1e9, bytes / 1e6);
    };
    char nm[160];
    const size_t n4 = L / 4;
    for (int per : {2, 4, 8}) {
        snprintf(nm, sizeof nm, "max ldg grid=%dxSM", per);
        timeit(nm, 4.0 * L, [&](int k) { k_max<<<per * sms, 256>>>((const float4 *)g[k % S], n4, mx, 1); });
    }
    for (int per : {2, 4, 8}) {
        for (int h : {0, 1}) {
            snprintf(nm, sizeof nm, "qu ldg grid=%dxSM sthint=%d", per, h);
            timeit(nm, step_bytes, [&](int k) { k_qu<<<per * sms, 256>>>((const float4 *)g[k % S], c[k % S], (float4 *)o[k % S], n4, 0, h); });
        }
    }
    for (int R : {32768, 65536}) {
        for (int St : {2, 3, 4, 6}) {
            const size_t smem = (size_t)St * R + 2 * St * 8 + 64;
            if (smem > 220 * 1024) continue;
            CK(cudaFuncSetAttribute(k_qu_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            snprintf(nm, sizeof nm, "qu tma R=%dK S=%d", R / 1024, St);
            timeit(nm, step_bytes, [&](int k) { k_qu_tma<<<sms, 288, smem>>>((const uint8_t *)g[k % S], c[k % S], (float4 *)o[k % S], 4 * L, R, St, 0); });
        }
    }
    for (int per : {4, 8}) {
        snprintf(nm, sizeof nm, "pair max(4xSM) + qu ldg rev grid=%dxSM", per);
        timeit(nm, step_bytes, [&](int k) {
            k_max<<<4 * sms, 256>>>((const float4 *)g[k % S], n4, mx, 1);
            k_qu<<<per * sms, 256>>>((const float4 *)g[k % S], c[k % S], (float4 *)o[k % S], n4, 1, 1);
        });
        snprintf(nm, sizeof nm, "pair max(4xSM) + qu ldg fwd grid=%dxSM", per);
        timeit(nm, step_bytes, [&](int k) {
            k_max<<<4 * sms, 256>>>((const float4 *)g[k % S], n4, mx, 1);
            k_qu<<<per * sms, 256>>>((const float4 *)g[k % S], c[k % S], (float4 *)o[k % S], n4, 0, 1);
        });
    }
    {
        const int R = 32768, St = 4;
        const size_t smem = (size_t)St * R + 2 * St * 8 + 64;
        CK(cudaFuncSetAttribute(k_qu_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        timeit("pair max(4xSM) + qu tma rev R=32K S=4", step_bytes, [&](int k) {
            k_max<<<4 * sms, 256>>>((const float4 *)g[k % S], n4, mx, 1);
            k_qu_tma<<<sms, 288, smem>>>((const uint8_t *)g[k % S], c[k % S], (float4 *)o[k % S], 4 * L, R, St, 1);
        });
    }
    return 0;
}
