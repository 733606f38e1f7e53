// mma_bench.cu — cycles per tcgen05.mma (kind::f16, SS operands, 128B swizzle) on this GPU,
// for M = 128, several N, with the K-steps accumulating into one TMEM tile (dependent) or
// spread over independent tiles.  Diagnostics only (tools/).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

template <int N, int M = 128, int MODE = 0>  // MODE 0: SS, 1: TS (A in TMEM), 2: tcgen05.cp 128x256b only
__global__ void k_mma(int iters, int nacc, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t sbB = sa + 16384;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)));
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
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t a = desc_sw128(sa, 16, 1024);
        const uint64_t b = desc_sw128(sbB, 16, 1024);
        const uint32_t barp = (uint32_t)__cvta_generic_to_shared(&bar);
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
            const uint32_t acc = i >= nacc ? 1u : 0u;
            if (MODE == 0)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                             ::"r"(d), "l"(a + ((i & 3) * 2)), "l"(b + ((i & 3) * 2)), "r"(idesc), "r"(acc));
            else if (MODE == 1)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(d), "r"(tmem + 256 + (uint32_t)((i & 3) * 8)), "l"(b + ((i & 3) * 2)), "r"(idesc), "r"(acc));
            else
                asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 256 + (uint32_t)((i & 3) * 8)), "l"(a + ((i & 3) * 2)));
        }
        unsigned long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(barp));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(barp));
        unsigned long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    unsigned long long h[2];
    const int iters = 4096;
    auto run = [&](auto kern, int n, int nacc) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        kern<<<1, 128, 65536>>>(iters, nacc, d);
        kern<<<1, 128, 65536>>>(iters, nacc, d);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        printf("N=%3d independent accumulators=%d: issue %.1f cyc/mma, complete %.1f cyc/mma %s\n", n, nacc,
               (double)h[0] / iters, (double)h[1] / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    printf("SS M=128:\n");
    run(k_mma<16>, 16, 1);
    run(k_mma<256>, 256, 1);
    printf("SS M=64:\n");
    run(k_mma<16, 64>, 16, 1);
    run(k_mma<64, 64>, 64, 1);
    printf("TS M=128 (A in TMEM):\n");
    run(k_mma<16, 128, 1>, 16, 1);
    run(k_mma<16, 128, 1>, 16, 4);
    run(k_mma<64, 128, 1>, 64, 1);
    run(k_mma<256, 128, 1>, 256, 1);
    printf("tcgen05.cp 128x256b (4 KB smem -> tmem):\n");
    run(k_mma<16, 128, 2>, 16, 1);
    return 0;
}
