// mma_bench4.cu — cost of the fused kernel's per-item tcgen05 issue pattern (MMAs + commits)
// in isolation, and with other warps loading shared memory concurrently.  Diagnostics only.
//   pattern 0: 4 x MMA(M128,N16)                                  (S^T of one d=64 chunk)
//   pattern 1: 4 x MMA(M128,N16) + 1 commit
//   pattern 2: 4 x MMA(M128,N16) + 3 commits
//   pattern 3: 4 x MMA(M128,N16) + 3 commits + 2 x MMA(M64,N16,MN-major A) + 2 commits (batched item)
//   pattern 4: 8 x MMA(M128,N16) + 2 commits + 8 x MMA(M128,N16,MN-major A) + 2 commits (arxiv chunk)
//   pattern 5: 4 x MMA(M64,N16) + 3 commits + 2 x MMA(M64,N16,MN-major) + 2 commits
// stress: 0 none, 1 = 8 warps of st.shared.v4 in a loop, 2 = 8 warps of cp.async 16 B from global
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
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(t), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                 ::"r"(bar) : "memory");
}
__host__ __device__ constexpr uint32_t idesc(uint32_t amn, uint32_t bmn, uint32_t M, uint32_t N) {
    return (1u << 4) | (amn << 15) | (bmn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int PAT, int STRESS>
__global__ void k(int outer, unsigned long long* out, const int4* g) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bars[8];
    __shared__ volatile int stop;
    const uint32_t sa = ((uint32_t)__cvta_generic_to_shared(smem) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        stop = 0;
        for (int i = 0; i < 8; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        auto bar = [&](int i) { return (uint32_t)__cvta_generic_to_shared(&bars[i]); };
        const uint64_t dK = desc_sw128(sa, 16, 1024);
        const uint64_t dQ = desc_sw128(sa + 65536, 16, 1024);
        const uint64_t dV = desc_sw128(sa, 1024, 1024);
        const uint64_t dP = desc_sw128(sa + 65536 + 8192, 4096, 256);
        unsigned long long t0 = clock64();
        for (int o = 0; o < outer; ++o) {
            const uint32_t tb = (o & 3) * 16;
            if (PAT == 0 || PAT == 1 || PAT == 2 || PAT == 3) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma(tmem + tb, dK + kk * 2, dQ + kk * 2, idesc(0, 0, 128, 16), kk > 0);
                if (PAT >= 1) commit(bar(0));
                if (PAT >= 2) { commit(bar(1)); commit(bar(2)); }
                if (PAT == 3) {
#pragma unroll
                    for (int st = 0; st < 2; ++st) mma(tmem + 64 + tb, dV + st * 128, dP + st * 32, idesc(1, 1, 64, 16), st > 0);
                    commit(bar(3));
                    commit(bar(4));
                }
            } else if (PAT == 4) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mma(tmem + tb, dK + kk * 2, dQ + kk * 2, idesc(0, 0, 128, 16), kk > 0);
                commit(bar(0));
                commit(bar(1));
#pragma unroll
                for (int st = 0; st < 8; ++st) mma(tmem + 64 + tb, dV + st * 128, dP + st * 32, idesc(1, 1, 128, 16), st > 0);
                commit(bar(3));
                commit(bar(4));
            } else if (PAT == 5) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) mma(tmem + tb, dK + kk * 2, dQ + kk * 2, idesc(0, 0, 64, 16), kk > 0);
                commit(bar(0));
                commit(bar(1));
                commit(bar(2));
#pragma unroll
                for (int st = 0; st < 2; ++st) mma(tmem + 64 + tb, dV + st * 128, dP + st * 32, idesc(1, 1, 64, 16), st > 0);
                commit(bar(3));
                commit(bar(4));
            }
        }
        unsigned long long t1 = clock64();
        commit(bar(5));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bars[5])));
        unsigned long long t2 = clock64();
        if (threadIdx.x == 0) {
            out[2 * blockIdx.x] = t1 - t0;
            out[2 * blockIdx.x + 1] = t2 - t0;
            stop = 1;
        }
    } else if (STRESS == 1) {
        // shared-memory store traffic into the upper 64 KB
        const uint32_t base = sa + 131072 + (threadIdx.x - 32) * 16;
        int it = 0;
        while (!stop) {
#pragma unroll 8
            for (int r = 0; r < 64; ++r)
                asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + ((r * 4096) & 65535)), "r"(it));
            ++it;
        }
    } else if (STRESS == 3 || STRESS == 4) {
        // mbarrier waiters that never succeed (phase 1 of bars[7] never completes), as the
        // kernel's mbar_wait: try_wait + global-timer read per retry (3) or try_wait only (4)
        const uint32_t b7 = (uint32_t)__cvta_generic_to_shared(&bars[7]);
        uint64_t acc = 0;
        while (!stop) {
            uint32_t ok;
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(b7));
            if (STRESS == 3) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); acc += t + ok; }
            else acc += ok;
        }
        if (acc == 12345) out[0] = acc;
    } else if (STRESS == 2) {
        const uint32_t base = sa + 131072 + (threadIdx.x - 32) * 16;
        size_t gi = (size_t)blockIdx.x * 4096 + threadIdx.x;
        while (!stop) {
#pragma unroll 8
            for (int r = 0; r < 64; ++r) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + ((r * 4096) & 65535)), "l"(g + (gi & ((1u << 24) - 1))));
                gi += 256 * 37;
            }
            asm volatile("cp.async.wait_all;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    unsigned long long* d;
    int4* g;
    cudaMalloc(&d, 16 * 512);
    cudaMalloc(&g, (size_t)16 << 24);
    cudaMemset(g, 0, (size_t)16 << 24);
    unsigned long long h[4];
    const int outer = 512;
    const int smem = 196608 + 1024;
    auto run = [&](auto kern, const char* nm, int threads) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<148, threads, smem>>>(outer, d, g);
        kern<<<148, threads, smem>>>(outer, d, g);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 4 * 8, cudaMemcpyDeviceToHost);
        printf("%-40s: issue %7.1f cyc/group, complete %7.1f cyc/group %s\n", nm, (double)h[0] / outer,
               (double)h[1] / outer, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    run(k<0, 0>, "4 MMA M128", 32);
    run(k<1, 0>, "4 MMA M128 + 1 commit", 32);
    run(k<2, 0>, "4 MMA M128 + 3 commits", 32);
    run(k<3, 0>, "batched item (4+2 MMA, 5 commits)", 32);
    run(k<5, 0>, "batched item, M64 MMA1", 32);
    run(k<4, 0>, "arxiv chunk (8+8 MMA, 4 commits)", 32);
    run(k<0, 1>, "4 MMA M128, st.shared stress", 288);
    run(k<3, 1>, "batched item, st.shared stress", 288);
    run(k<4, 1>, "arxiv chunk, st.shared stress", 288);
    run(k<3, 3>, "batched item, 8 spinners (timer)", 288);
    run(k<3, 3>, "batched item, 19 spinners (timer)", 640);
    run(k<3, 4>, "batched item, 19 spinners (no timer)", 640);
    run(k<4, 3>, "arxiv chunk, 19 spinners (timer)", 640);
    run(k<0, 2>, "4 MMA M128, cp.async stress", 288);
    run(k<3, 2>, "batched item, cp.async stress", 288);
    run(k<4, 2>, "arxiv chunk, cp.async stress", 288);
    return 0;
}
