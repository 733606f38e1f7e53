// gather_bench2.cu — gather throughput of the fused kernel's loader design alternatives, in the
// kernel's own shape: one persistent CTA per SM, a stream of 128-row chunks (K and V head slices of
// the plan's compacted columns, 8 lanes per 128-byte row), a ring of shared-memory tiles, and a
// consumer warp that releases each tile as soon as it has landed.  Diagnostics only.
//   mode 0: cp.async 16 B (LDGSTS), completion by cp.async.mbarrier.arrive.noinc
//   mode 1: LDG.128 into registers, then STS.128 into the swizzled tile, fence.proxy.async + arrive
// pf > 0: a prefetch warp issues prefetch.global.L2 for every row of chunk i + pf (per CTA stream)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}

constexpr int kRows = 128, kTile = 2 * kRows * 128;  // K + V, d = 64 fp16 (128-byte rows)
constexpr int kIdx = 24;  // chunk-id ring (the kernel's slots): filled ahead by the index/prefetch warp

__device__ __forceinline__ void gather4(uint32_t dst, const void* tmap, uint32_t bar, int32_t x, int4 r) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        ::"r"(dst), "l"(tmap), "r"(bar), "r"(x), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w) : "memory");
}

template <int MODE, int NL>
__global__ void __launch_bounds__(32 * (NL + 2), 1)
k_bench(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
        const int32_t* __restrict__ cols, int64_t n_chunks, int H, const uint8_t* __restrict__ K,
        const uint8_t* __restrict__ V, int ntiles, int pf, uint32_t* __restrict__ sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[2 * 16 + kIdx];
    __shared__ int32_t ids[kIdx][kRows];
    __shared__ volatile int32_t consumed;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars);
    auto full = [&](int t) { return b0 + 8u * t; };
    auto empty = [&](int t) { return b0 + 8u * (16 + t); };
    auto idxf = [&](int s) { return b0 + 8u * (32 + s); };
    if (threadIdx.x == 0) {
        consumed = 0;
        for (int t = 0; t < ntiles; ++t) {
            mbar_init(full(t), MODE == 2 ? NL : 32 * NL);
            mbar_init(empty(t), 1);
        }
        for (int s = 0; s < kIdx; ++s) mbar_init(idxf(s), 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ldb = (int64_t)H * 128;
    const int64_t mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto chunk_of = [&](int64_t i) { return blockIdx.x + i * gridDim.x; };
    if (warp == NL + 1) {  // index + prefetch warp: stages chunk ids ahead, prefetches rows to L2
        // one 16-byte load of 4 ids per lane per chunk, software-pipelined 4 chunks deep
        auto ld_ids = [&](int64_t i) -> int4 {
            if (i >= mine) return make_int4(0, 0, 0, 0);
            const int64_t c = chunk_of(i);
            return __ldg(reinterpret_cast<const int4*>(cols + (c / H) * kRows) + lane);
        };
        int4 q0 = ld_ids(0), q1 = ld_ids(1), q2 = ld_ids(2), q3 = ld_ids(3);
        const int64_t lead = pf > 0 ? (pf < kIdx ? pf : kIdx) : kIdx;
        for (int64_t i = 0; i < mine; ++i) {
            const int4 cur = q0;
            q0 = q1; q1 = q2; q2 = q3; q3 = ld_ids(i + 4);
            while (consumed < i - lead + 1) __nanosleep(64);
            const int h = (int)(chunk_of(i) % H);
            const int s = (int)(i % kIdx);
            reinterpret_cast<int4*>(ids[s])[lane] = cur;
            if (pf > 0) {
                const int jj[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(K + (int64_t)jj[u] * ldb + h * 128));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(V + (int64_t)jj[u] * ldb + h * 128));
                }
            }
            mbar_arrive(idxf(s));
        }
        return;
    }
    if (warp == NL) {  // consumer: release each tile once it landed
        for (int64_t i = 0; i < mine; ++i) {
            const int t = (int)(i % ntiles);
            mbar_wait(full(t), (i / ntiles) & 1);
            if (lane == 0) { mbar_arrive(empty(t)); consumed = (int32_t)(i + 1); }
        }
        return;
    }
    // loaders: warp w handles row ops w, w + NL, ... (4 rows per op: 8 lanes x 16 B per row)
    const int piece = lane & 7, rsub = lane >> 3;
    if (MODE == 7) {
        // LDG + STS, software-pipelined 3 chunks deep: the loads of chunk i + 3 are issued as soon
        // as chunk i's registers are stored
        constexpr int kOps = (kRows / 4 + NL - 1) / NL;
        uint4 kA[kOps], vA[kOps], kB[kOps], vB[kOps], kC[kOps], vC[kOps];
        auto issue = [&](int64_t j, uint4 (&kk)[kOps], uint4 (&vv)[kOps]) {
            if (j >= mine) return;
            const int s = (int)(j % kIdx);
            mbar_wait(idxf(s), (j / kIdx) & 1);
            const int h = (int)(chunk_of(j) % H);
#pragma unroll
            for (int q = 0; q < kOps; ++q) {
                const int op = warp + q * NL;
                if (op < kRows / 4) {
                    const int64_t jj = ids[s][op * 4 + rsub];
                    kk[q] = __ldg(reinterpret_cast<const uint4*>(K + jj * ldb + h * 128 + piece * 16));
                    vv[q] = __ldg(reinterpret_cast<const uint4*>(V + jj * ldb + h * 128 + piece * 16));
                }
            }
        };
        auto store = [&](int64_t j, uint4 (&kk)[kOps], uint4 (&vv)[kOps]) {
            if (j >= mine) return;
            const int t = (int)(j % ntiles);
            if (j >= ntiles) mbar_wait(empty(t), ((j / ntiles) & 1) ^ 1);
            const uint32_t kt = (uint32_t)__cvta_generic_to_shared(smem + (size_t)t * kTile);
            const uint32_t vt = kt + kRows * 128;
#pragma unroll
            for (int q = 0; q < kOps; ++q) {
                const int op = warp + q * NL;
                if (op < kRows / 4) {
                    const int r = op * 4 + rsub;
                    const uint32_t o = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(kt + o), "r"(kk[q].x), "r"(kk[q].y),
                                 "r"(kk[q].z), "r"(kk[q].w) : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(vt + o), "r"(vv[q].x), "r"(vv[q].y),
                                 "r"(vv[q].z), "r"(vv[q].w) : "memory");
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(full(t));
        };
        issue(0, kA, vA);
        issue(1, kB, vB);
        issue(2, kC, vC);
        for (int64_t i = 0; i < mine; i += 3) {
            store(i, kA, vA);
            issue(i + 3, kA, vA);
            store(i + 1, kB, vB);
            issue(i + 4, kB, vB);
            store(i + 2, kC, vC);
            issue(i + 5, kC, vC);
        }
        return;
    }
    uint32_t acc = 0;
    for (int64_t i = 0; i < mine; ++i) {
        const int t = (int)(i % ntiles);
        if (i >= ntiles) mbar_wait(empty(t), ((i / ntiles) & 1) ^ 1);
        const int s = (int)(i % kIdx);
        mbar_wait(idxf(s), (i / kIdx) & 1);
        const int64_t c = chunk_of(i);
        const int h = (int)(c % H);
        const uint32_t kt = (uint32_t)__cvta_generic_to_shared(smem + (size_t)t * kTile);
        const uint32_t vt = kt + kRows * 128;
        if (MODE == 2 || MODE == 3) {
            // TMA tile::gather4: one elected lane per warp, 4 rows (512 B) per instruction;
            // MODE 3: K by TMA, V by cp.async
            if (lane == 0) {
                if (MODE == 2) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(t)),
                                            "r"(2 * (kRows / NL) * 128) : "memory");
                else asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(full(t)),
                                  "r"((kRows / NL) * 128) : "memory");
                for (int op = warp; op < kRows / 4; op += NL) {
                    const int4 r = reinterpret_cast<const int4*>(ids[s])[op];
                    const uint32_t o = (uint32_t)(op >> 1) * 1024 + (uint32_t)(op & 1) * 512;
                    gather4(kt + o, &tk, full(t), h * 64, r);
                    if (MODE == 2) gather4(vt + o, &tv, full(t), h * 64, r);
                }
            }
            if (MODE == 3) {
                for (int op = warp; op < kRows / 4; op += NL) {
                    const int r = op * 4 + rsub;
                    const int64_t j = ids[s][r];
                    const uint32_t o = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vt + o), "l"(V + j * ldb + h * 128 + piece * 16) : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(t)) : "memory");
            }
        } else if (MODE >= 5) {
            // hybrid: warps [0, NC) cp.async rows [0, RS), warps [NC, NL) LDG + STS rows [RS, 128)
            constexpr int NC = MODE == 5 ? NL * 3 / 4 : NL / 2;
            constexpr int RS = (kRows * NC / NL) / 4 * 4;
            if (warp < NC) {
                for (int op = warp; op < RS / 4; op += NC) {
                    const int r = op * 4 + rsub;
                    const int64_t j = ids[s][r];
                    const uint32_t o = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(kt + o), "l"(K + j * ldb + h * 128 + piece * 16) : "memory");
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vt + o), "l"(V + j * ldb + h * 128 + piece * 16) : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(t)) : "memory");
            } else {
                constexpr int NLD = NL - NC;
                constexpr int kOps = ((kRows - RS) / 4 + NLD - 1) / NLD;
                uint4 kv[kOps], vv[kOps];
                uint32_t off[kOps];
                bool okk[kOps];
#pragma unroll
                for (int q = 0; q < kOps; ++q) {
                    const int op = RS / 4 + (warp - NC) + q * NLD;
                    okk[q] = op < kRows / 4;
                    const int r = okk[q] ? op * 4 + rsub : 0;
                    const int64_t j = ids[s][r];
                    off[q] = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                    if (okk[q]) {
                        kv[q] = __ldg(reinterpret_cast<const uint4*>(K + j * ldb + h * 128 + piece * 16));
                        vv[q] = __ldg(reinterpret_cast<const uint4*>(V + j * ldb + h * 128 + piece * 16));
                    }
                }
#pragma unroll
                for (int q = 0; q < kOps; ++q)
                    if (okk[q]) {
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(kt + off[q]), "r"(kv[q].x), "r"(kv[q].y),
                                     "r"(kv[q].z), "r"(kv[q].w) : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(vt + off[q]), "r"(vv[q].x), "r"(vv[q].y),
                                     "r"(vv[q].z), "r"(vv[q].w) : "memory");
                    }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(full(t));
            }
        } else if (MODE == 4) {
            for (int op = warp; op < kRows / 4; op += NL) {
                const int r = op * 4 + rsub;
                const int64_t j = ids[s][r];
                const uint32_t o = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(kt + o), "l"(K + j * ldb + h * 128 + piece * 16) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(vt + o), "l"(V + j * ldb + h * 128 + piece * 16) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(t)) : "memory");
        } else if (MODE == 0) {
            for (int op = warp; op < kRows / 4; op += NL) {
                const int r = op * 4 + rsub;
                const int64_t j = ids[s][r];
                const uint32_t o = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(kt + o), "l"(K + j * ldb + h * 128 + piece * 16) : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vt + o), "l"(V + j * ldb + h * 128 + piece * 16) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(t)) : "memory");
        } else {
            constexpr int kOps = kRows / 4 / NL;  // row ops per warp per chunk
            uint4 kv[kOps], vv[kOps];
            uint32_t off[kOps];
#pragma unroll
            for (int q = 0; q < kOps; ++q) {
                const int r = (warp + q * NL) * 4 + rsub;
                const int64_t j = ids[s][r];
                off[q] = (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128 + (uint32_t)((piece ^ (r & 7)) << 4);
                kv[q] = __ldg(reinterpret_cast<const uint4*>(K + j * ldb + h * 128 + piece * 16));
                vv[q] = __ldg(reinterpret_cast<const uint4*>(V + j * ldb + h * 128 + piece * 16));
            }
#pragma unroll
            for (int q = 0; q < kOps; ++q) {
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(kt + off[q]), "r"(kv[q].x), "r"(kv[q].y),
                             "r"(kv[q].z), "r"(kv[q].w) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(vt + off[q]), "r"(vv[q].x), "r"(vv[q].y),
                             "r"(vv[q].z), "r"(vv[q].w) : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(full(t));
        }
    }
    if (acc == 0x12345u) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int64_t g_nrows = 0;
static void make_map(CUtensorMap* m, const void* base, int H) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    cuuint64_t dims[2] = {(cuuint64_t)H * 64, (cuuint64_t)g_nrows};
    cuuint64_t str[1] = {(cuuint64_t)H * 64 * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, str, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}

template <int MODE, int NL>
static float run(const int32_t* cols, int64_t n_chunks, int H, const void* K, const void* V, int ntiles, int pf, int reps) {
    uint32_t* sink;
    cudaMalloc(&sink, 64);
    CUtensorMap tk, tv;
    make_map(&tk, K, H);
    make_map(&tv, V, H);
    const int smem = ntiles * kTile;
    cudaFuncSetAttribute(k_bench<MODE, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        k_bench<MODE, NL><<<148, 32 * (NL + 2), smem>>>(tk, tv, cols, n_chunks, H, (const uint8_t*)K, (const uint8_t*)V, ntiles, pf, sink);
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

extern "C" float gather_bench2(int mode, int nl, const int32_t* cols, int64_t n_chunks, int H, const void* K,
                               const void* V, int ntiles, int pf, int reps, int64_t n_rows) {
    g_nrows = n_rows;
    if (mode == 7 && nl == 16) return run<7, 16>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 7 && nl == 24) return run<7, 24>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 7 && nl == 8) return run<7, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 5 && nl == 8) return run<5, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 5 && nl == 12) return run<5, 12>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 6 && nl == 8) return run<6, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 6 && nl == 12) return run<6, 12>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 4 && nl == 4) return run<4, 4>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 4 && nl == 8) return run<4, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 0 && nl == 12) return run<0, 12>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 0 && nl == 16) return run<0, 16>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 2 && nl == 4) return run<2, 4>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 2 && nl == 8) return run<2, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 3 && nl == 4) return run<3, 4>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 3 && nl == 8) return run<3, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 0 && nl == 4) return run<0, 4>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 0 && nl == 8) return run<0, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 1 && nl == 4) return run<1, 4>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 1 && nl == 8) return run<1, 8>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    if (mode == 1 && nl == 16) return run<1, 16>(cols, n_chunks, H, K, V, ntiles, pf, reps);
    return -1.f;
}
