// mma_bench2.cu — issue cost of tcgen05.mma kind::f16 in straight-line code (no per-iteration
// integer work): REP unrolled MMAs with compile-time descriptor offsets, per N and M, and with
// 1 or 2 CTAs per SM issuing concurrently.  Diagnostics only (tools/).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)(1) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

template <int N, int M, int REP, int V = 0>
__global__ void k_mma(int outer, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sa = ((uint32_t)__cvta_generic_to_shared(smem) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x < 32) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t a = desc_sw128(sa);
        const uint64_t b = desc_sw128(sa + 32768);
        const uint32_t barp = (uint32_t)__cvta_generic_to_shared(&bar);
        unsigned long long t0 = clock64();
        for (int o = 0; o < outer; ++o) {
            if (V == 2) {
#pragma unroll
                for (int i = 0; i < REP; ++i) {
                    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff;\n\t@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;}"
                                 ::"r"(tmem), "l"(a + (uint64_t)((i & 3) * 2)), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc));
                }
            } else if (__builtin_expect(threadIdx.x == 0, 1)) {
#pragma unroll
                for (int i = 0; i < REP; ++i) {
                    const uint64_t off = V == 1 ? 0 : (uint64_t)((i & 3) * 2);
                    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                                 ::"r"(tmem), "l"(a + off), "l"(b + off), "r"(idesc));
                }
            }
            __syncwarp();
        }
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(barp));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(barp));
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) {
            out[2 * blockIdx.x] = t1 - t0;
            out[2 * blockIdx.x + 1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16 * 512);
    unsigned long long h[16];
    const int outer = 256, REP = 16;
    auto run = [&](auto kern, const char* nm, int ctas) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 66560);
        kern<<<ctas, 128, 66560>>>(outer, d);
        kern<<<ctas, 128, 66560>>>(outer, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        printf("%-14s ctas=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma %s\n", nm, ctas,
               (double)h[0] / (outer * REP), (double)h[1] / (outer * REP), e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    for (int ctas : {1, 296}) {
        run(k_mma<16, 128, REP, 0>, "M128 N16 v0", ctas);
        run(k_mma<16, 128, REP, 1>, "M128 N16 v1", ctas);
        run(k_mma<16, 128, REP, 2>, "M128 N16 v2", ctas);
        run(k_mma<16, 64, REP, 1>, "M64 N16 v1", ctas);
        run(k_mma<16, 64, REP, 2>, "M64 N16 v2", ctas);
        run(k_mma<64, 128, REP, 2>, "M128 N64 v2", ctas);
        run(k_mma<128, 128, REP, 2>, "M128 N128 v2", ctas);
    }
    return 0;
}
