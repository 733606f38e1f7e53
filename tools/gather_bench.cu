// gather_bench.cu — how fast can a B200 gather the K/V rows the fused 3S pass needs?
// Reads, for every (compacted column, head) of a plan, the 2 x d x 2-byte K and V rows,
// exactly the algorithmic gather traffic of the hot path, with three mechanisms:
//   0: LDG.128 into registers (XOR-reduced), full occupancy
//   1: cp.async 16 B into a per-warp shared-memory buffer
//   2: TMA tile::gather4 (box 64 x 1, 128B swizzle) into shared memory, one issuing lane per warp
// Diagnostics only (tools/); not part of the library.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void k_ldg(const int32_t* __restrict__ cols, int64_t W, int H, int D, const uint4* __restrict__ K,
                      const uint4* __restrict__ V, uint32_t* __restrict__ sink) {
    const int pieces = D * 2 / 16;  // 16-B pieces per (row, head)
    const int64_t total = W * H * pieces;
    const int64_t ld = (int64_t)H * pieces;
    uint32_t acc = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t / (H * pieces);
        const int rem = (int)(t - e * H * pieces);
        const int64_t j = __ldg(cols + e);
        const uint4 a = __ldg(K + j * ld + rem);
        const uint4 b = __ldg(V + j * ld + rem);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void k_cpasync(const int32_t* __restrict__ cols, int64_t W, int H, int D, const uint8_t* __restrict__ K,
                          const uint8_t* __restrict__ V, uint32_t* __restrict__ sink) {
    extern __shared__ __align__(16) uint8_t buf[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int pieces = D * 2 / 16;
    const int rows_per_op = 32 / pieces;
    const int64_t ldb = (int64_t)H * D * 2;
    // each warp owns 8 KB of smem split in 4 stages of 2 KB (K+V of rows_per_op*? rows)
    uint8_t* wb = buf + warp * 8192;
    const int64_t units = W * H;  // (entry, head)
    const int64_t gw = blockIdx.x * (int64_t)nwarps + warp, nw = (int64_t)gridDim.x * nwarps;
    int stage = 0;
    for (int64_t u0 = gw * rows_per_op; u0 < units; u0 += nw * rows_per_op) {
        const int64_t u = u0 + lane / pieces;
        if (u < units) {
            const int64_t e = u / H;
            const int h = (int)(u - e * H);
            const int64_t j = __ldg(cols + e);
            const uint32_t dk = (uint32_t)__cvta_generic_to_shared(wb + stage * 2048 + lane * 16);
            const uint32_t dv = dk + 1024;
            const uint8_t* src_k = K + j * ldb + h * D * 2 + (lane % pieces) * 16;
            const uint8_t* src_v = V + j * ldb + h * D * 2 + (lane % pieces) * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk), "l"(src_k) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dv), "l"(src_v) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 3;" ::: "memory");
        stage = (stage + 1) & 3;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (reinterpret_cast<uint32_t*>(wb)[lane] == 0x12345678u) sink[0] = 1;
}

__global__ void k_tma(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                      const int32_t* __restrict__ cols, int64_t W, int H, int D, uint32_t* __restrict__ sink) {
    extern __shared__ __align__(1024) uint8_t buf[];
    __shared__ __align__(8) uint64_t bars[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int P = D / 64;
    // warp w: 4 stages x (K,V) x 4 rows x P panels x 128 B
    const int stage_bytes = 2 * 4 * P * 128;
    uint8_t* wb = buf + warp * 4 * stage_bytes;
    if (lane == 0)
        for (int s = 0; s < 4; ++s) {
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[(warp * 4 + s) % 16]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (nwarps * 4 > 16) return;
    const int64_t units4 = (W + 3) / 4 * H;  // groups of 4 entries x head
    const int64_t gw = blockIdx.x * (int64_t)nwarps + warp, nw = (int64_t)gridDim.x * nwarps;
    uint32_t phase[4] = {0, 0, 0, 0};
    int stage = 0;
    int64_t issued = 0;
    for (int64_t g = gw; g < units4; g += nw) {
        const int64_t e4 = (g / H) * 4;
        const int h = (int)(g - (g / H) * H);
        int32_t r[4];
        for (int q = 0; q < 4; ++q) r[q] = __ldg(cols + min(e4 + q, W - 1));
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp * 4 + stage]);
        if (lane == 0) {
            if (issued >= 4) {
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                                 : "=r"(ok) : "r"(bar), "r"(phase[stage]) : "memory");
                phase[stage] ^= 1;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * 4 * P * 128) : "memory");
            for (int pp = 0; pp < P; ++pp) {
                const uint32_t dk = (uint32_t)__cvta_generic_to_shared(wb + stage * stage_bytes + pp * 512);
                const uint32_t dv = dk + 4 * P * 128;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                    ::"r"(dk), "l"(&tk), "r"(bar), "r"(h * D + 64 * pp), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                    ::"r"(dv), "l"(&tv), "r"(bar), "r"(h * D + 64 * pp), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
            }
        }
        ++issued;
        stage = (stage + 1) & 3;
    }
    if (lane == 0)
        for (int s = 0; s < 4 && s < issued; ++s) {
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp * 4 + s]);
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(bar), "r"(phase[s]) : "memory");
        }
    if (wb[lane] == 0x7f && wb[lane + 1] == 0x13) sink[0] = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" float gather_bench(int mode, const int32_t* cols, int64_t W, int H, int D, const void* K, const void* V,
                              int64_t n_rows, int grid, int block, int reps) {
    uint32_t* sink;
    cudaMalloc(&sink, 64);
    CUtensorMap tk, tv;
    if (mode == 2) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        cuuint64_t dims[2] = {(cuuint64_t)H * D, (cuuint64_t)n_rows};
        cuuint64_t str[1] = {(cuuint64_t)H * D * 2};
        cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
        ((EncodeFn)fn)(&tk, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(K), dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        ((EncodeFn)fn)(&tv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(V), dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    int smem = mode == 1 ? (block / 32) * 8192 : (mode == 2 ? (block / 32) * 4 * 2 * 4 * (D / 64) * 128 + 1024 : 0);
    if (mode == 1) cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (mode == 2) cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        if (mode == 0) k_ldg<<<grid, block>>>(cols, W, H, D, (const uint4*)K, (const uint4*)V, sink);
        if (mode == 1) k_cpasync<<<grid, block, smem>>>(cols, W, H, D, (const uint8_t*)K, (const uint8_t*)V, sink);
        if (mode == 2) k_tma<<<grid, block, smem>>>(tk, tv, cols, W, H, D, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    cudaFree(sink);
    return best;
}
