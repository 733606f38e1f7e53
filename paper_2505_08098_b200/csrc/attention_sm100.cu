// attention_sm100.cu — the fused 3S kernel for B200 (sm_100a).
//
// Computes, per row window k (16 query rows) and head h, Alg.1 of the paper
// re-designed for Blackwell:
//
//   * work items (k, h) in LPT order from a persistent queue: one atomic per item;
//   * warp 0 (producer): TMA-loads Q_w (16 x d, Alg.1 l.5) and, per chunk of up to 128
//     compacted columns (sptd, l.7), gathers the K and V rows with cp.async.bulk.tensor
//     tile::gather4 (l.8) into a variable-size shared-memory ring (128B-swizzled tiles);
//   * warp 1 (MMA issuer, one thread): swap-AB contractions on tcgen05 with TMEM accumulators
//       MMA1  S^T[C x 16]  = K_c[C x d] . Q_w^T        (SDDMM, l.13; M = 128, N = 16)
//       MMA2  O^T[d x 16]  = V_c^T[d x C] . P^T[C x 16] (SpMM,  l.22; M = d,   N = 16)
//     S^T lane p is compacted column p, so the 16-bit plan mask of that column is the
//     bitmap row (l.14) of exactly one thread;
//   * warps 2-5 (128 threads): tcgen05.ld S^T, mask to -inf, chunk row max by warp
//     shuffles + a 4-warp combine, online softmax in fp32 with exp2 (l.16-18), P cast to the
//     input dtype into shared memory (l.19), then fold the chunk's O^T into fp32 registers
//     with the running rescale (l.21), and at the last chunk write O = O / l (l.24; rows with
//     l = 0 -> 0, reading c4).
//
// Everything between the gathers and the O store stays on chip.  No atomics on
// the data path: results are bitwise deterministic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "internal.h"
#include "sm100.cuh"

namespace f3s {
namespace {

using namespace sm100;

template <int D>
struct Cfg {
    static constexpr int P = D / 64;                 // 128-byte panels per gathered row of one head
    static constexpr int kGroupBytes = 1024 * P;     // 8 gathered rows (one swizzle atom per panel)
    static constexpr int kMaxRows = 128;             // chunk = up to 128 compacted columns (MMA1 M)
    static constexpr int kRingBytes = D == 128 ? 160 * 1024 : 80 * 1024;
    static constexpr int kNS = 16;                   // chunk slots (descriptor + barriers)
    static constexpr int kNQ = 4;                    // Q tile slots
    static constexpr int kQBytes = 16 * D * 2;
    static constexpr int kPBytes = 16 * kMaxRows * 2;
    static constexpr int kPad = D == 128 ? 8 * 1024 : 0;  // MMA1 may read past a short tile (masked lanes)
    static constexpr int oRing = 0;
    static constexpr int oQ = oRing + kRingBytes;
    static constexpr int oP = oQ + kNQ * kQBytes;
    static constexpr int oRed = oP + 2 * kPBytes + kPad;  // float [2][4][16] chunk row-max partials
    static constexpr int oLred = oRed + 2 * 4 * 16 * 4;   // float [4][16] row-sum partials
    static constexpr int oDesc = oLred + 4 * 16 * 4;      // ChunkDesc [kNS]
    static constexpr int oReg = oDesc + kNS * 32;         // int2 [kNS] ring regions
    static constexpr int kNumBars = 3 * kNS + 2 * kNQ + 6;
    static constexpr int oBar = oReg + kNS * 8;
    static constexpr int oTmem = oBar + kNumBars * 8;
    static constexpr int kSmemBytes = oTmem + 16 + 1024;  // + slack for 1024-byte alignment
    static constexpr int kCtasPerSm = D == 128 ? 1 : 2;
    static constexpr int kThreads = 192;
    static_assert(kRingBytes >= 2 * 2 * (kMaxRows / 8) * kGroupBytes, "ring must hold two full chunks");
    static_assert(oQ + kNQ * kQBytes + 2 * kPBytes + kPad >= kRingBytes + 12 * kGroupBytes, "over-read pad");
};

// barrier indices
template <int D> struct Bars {
    using C = Cfg<D>;
    __host__ __device__ static constexpr int kfull(int s) { return s; }
    __host__ __device__ static constexpr int vfull(int s) { return C::kNS + s; }
    __host__ __device__ static constexpr int empty(int s) { return 2 * C::kNS + s; }
    __host__ __device__ static constexpr int qfull(int q) { return 3 * C::kNS + q; }
    __host__ __device__ static constexpr int qempty(int q) { return 3 * C::kNS + C::kNQ + q; }
    __host__ __device__ static constexpr int sfull(int b) { return 3 * C::kNS + 2 * C::kNQ + b; }
    __host__ __device__ static constexpr int pfull(int b) { return 3 * C::kNS + 2 * C::kNQ + 2 + b; }
    __host__ __device__ static constexpr int ofull(int b) { return 3 * C::kNS + 2 * C::kNQ + 4 + b; }
};

struct __align__(16) ChunkDesc {
    int32_t rw;        // row window k
    int32_t head;      // head h
    int32_t col_base;  // index of the chunk's first compacted column in cols/masks
    int32_t rows;      // valid compacted columns in this chunk (0 for an empty RW, -1 = stop)
    int32_t ring_off;  // byte offset of the K tile in the ring (V tile follows)
    int32_t qslot;
    int32_t flags;     // bit0 first chunk of item, bit1 last chunk, bit2 Q-slot phase
    int32_t ralloc;    // rows allocated (multiple of 16)
};

// Transposing butterfly: 16 per-row values in each of 32 lanes -> lane l holds the
// reduction over the warp for row (l >> 1) & 15.  16 shuffles.
template <class Op>
__device__ __forceinline__ float rowreduce16(const float (&v)[16], int lane, Op op) {
    float a[8], b[4], c[2];
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const float mine = u16 ? v[r + 8] : v[r], send = u16 ? v[r] : v[r + 8];
        a[r] = op(mine, __shfl_xor_sync(0xffffffffu, send, 16));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const float mine = u8 ? a[r + 4] : a[r], send = u8 ? a[r] : a[r + 4];
        b[r] = op(mine, __shfl_xor_sync(0xffffffffu, send, 8));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const float mine = u4 ? b[r + 2] : b[r], send = u4 ? b[r] : b[r + 2];
        c[r] = op(mine, __shfl_xor_sync(0xffffffffu, send, 4));
    }
    const float mine = u2 ? c[1] : c[0], send = u2 ? c[0] : c[1];
    const float d = op(mine, __shfl_xor_sync(0xffffffffu, send, 2));
    return op(d, __shfl_xor_sync(0xffffffffu, d, 1));
}
struct OpMax { __device__ float operator()(float a, float b) const { return fmaxf(a, b); } };
struct OpAdd { __device__ float operator()(float a, float b) const { return a + b; } };

template <typename T> __device__ __forceinline__ uint16_t to_bits(float x);
template <> __device__ __forceinline__ uint16_t to_bits<__half>(float x) { return __half_as_ushort(__float2half_rn(x)); }
template <> __device__ __forceinline__ uint16_t to_bits<__nv_bfloat16>(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

template <int D, typename T>
__global__ void __launch_bounds__(Cfg<D>::kThreads, Cfg<D>::kCtasPerSm)
k_f3s_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, const int32_t* __restrict__ rw_ptr,
            const int32_t* __restrict__ cols, const uint16_t* __restrict__ masks, const int32_t* __restrict__ order,
            int32_t* __restrict__ counter, int32_t n_items, int32_t H, int32_t n_rows, float* __restrict__ O,
            float scale_log2) {
    using C = Cfg<D>;
    using B = Bars<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto bar = [&](int i) -> uint32_t { return sb + C::oBar + 8u * i; };
    ChunkDesc* descs = reinterpret_cast<ChunkDesc*>(smem + C::oDesc);

    // ---- setup -------------------------------------------------------------------------------
    // Ring bytes that no gather overwrites are read by MMA2 (rows between the last gathered
    // 4-row group and the 16-row MMA step, weighted by P = 0): they must be finite, so zero them.
    for (int i = threadIdx.x; i < C::kRingBytes / 16; i += blockDim.x)
        reinterpret_cast<int4*>(smem + C::oRing)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kNS; ++s) {
            mbar_init(bar(B::kfull(s)), 1);
            mbar_init(bar(B::vfull(s)), 1);
            mbar_init(bar(B::empty(s)), 1);
        }
        for (int q = 0; q < C::kNQ; ++q) {
            mbar_init(bar(B::qfull(q)), 1);
            mbar_init(bar(B::qempty(q)), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar(B::sfull(b)), 1);
            mbar_init(bar(B::pfull(b)), 128);
            mbar_init(bar(B::ofull(b)), 1);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
    }
    if (warp == 1) {
        tmem_alloc<64>(sb + C::oTmem);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::oTmem);

    if (warp == 0) {
        // ===== producer: work queue, Q tiles, K/V gathers ======================================
        const uint64_t pol = policy_evict_normal();
        int2* reg = reinterpret_cast<int2*>(smem + C::oReg);
        int32_t seq = 0, tail = 0, qseq = 0;
        uint32_t head = 0;
        for (;;) {
            int32_t item = 0;
            if (lane == 0) item = atomicAdd(counter, 1);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= n_items) break;
            const int32_t kq = item / H;
            const int32_t h = item - kq * H;
            const int32_t k = __ldg(order + kq);
            const int32_t cb = __ldg(rw_ptr + k), w = __ldg(rw_ptr + k + 1) - cb;
            const int qs = qseq % C::kNQ;
            const uint32_t qph = (qseq / C::kNQ) & 1;
            mbar_wait(bar(B::qempty(qs)), qph ^ 1);
            if (lane == 0) {
                mbar_arrive_expect_tx(bar(B::qfull(qs)), C::kQBytes);
#pragma unroll
                for (int pp = 0; pp < C::P; ++pp)
                    tma_load_2d(sb + C::oQ + qs * C::kQBytes + pp * 2048, &tmQ, bar(B::qfull(qs)), h * D + 64 * pp,
                                16 * k);
            }
            const int nch = w > 0 ? (w + C::kMaxRows - 1) / C::kMaxRows : 1;
            for (int j = 0; j < nch; ++j) {
                const int rows = w > 0 ? min(C::kMaxRows, w - C::kMaxRows * j) : 0;
                const int ralloc = rows > 0 ? ((rows + 15) & ~15) : 0;
                const uint32_t tile = (uint32_t)(ralloc / 8) * C::kGroupBytes;
                const uint32_t bytes = 2 * tile;
                // the slot's previous chunk must be retired (descriptor and barriers reused)
                while (tail <= seq - C::kNS) {
                    mbar_wait(bar(B::empty(tail % C::kNS)), (tail / C::kNS) & 1);
                    ++tail;
                }
                uint32_t off = 0;
                if (bytes > 0) {
                    off = head + bytes <= (uint32_t)C::kRingBytes ? head : 0;
                    for (;;) {  // retire the oldest chunks until [off, off+bytes) is free
                        bool ov = false;
                        for (int t = tail; t < seq; ++t) {
                            const int2 r = reg[t % C::kNS];
                            if (r.y > r.x && (int)off < r.y && (int)(off + bytes) > r.x) { ov = true; break; }
                        }
                        if (!ov) break;
                        mbar_wait(bar(B::empty(tail % C::kNS)), (tail / C::kNS) & 1);
                        ++tail;
                    }
                    head = off + bytes;
                }
                const int s = seq % C::kNS;
                __syncwarp();
                if (lane == 0) {
                    reg[s] = make_int2((int)off, (int)(off + bytes));
                    ChunkDesc dsc;
                    dsc.rw = k;
                    dsc.head = h;
                    dsc.col_base = cb + C::kMaxRows * j;
                    dsc.rows = rows;
                    dsc.ring_off = (int)off;
                    dsc.qslot = qs;
                    dsc.flags = (j == 0 ? 1 : 0) | (j == nch - 1 ? 2 : 0) | (int)(qph << 2);
                    dsc.ralloc = ralloc;
                    descs[s] = dsc;
                }
                __syncwarp();
                const uint32_t kfb = bar(B::kfull(s)), vfb = bar(B::vfull(s));
                const int ng = (rows + 3) >> 2;  // gather4 groups
                if (lane == 0) {
                    if (rows > 0) {
                        mbar_arrive_expect_tx(kfb, (uint32_t)ng * 512u * C::P);
                        mbar_arrive_expect_tx(vfb, (uint32_t)ng * 512u * C::P);
                    } else {
                        mbar_arrive(kfb);
                        mbar_arrive(vfb);
                    }
                }
                __syncwarp();
                if (lane < ng) {
                    // rows past the end of the chunk repeat its last column: finite data,
                    // masked out of the softmax and weighted 0 in the SpMM
                    const int32_t* cp = cols + cb + C::kMaxRows * j;
                    const int r0 = 4 * lane, last = rows - 1;
                    const int32_t i0 = __ldg(cp + min(r0, last)), i1 = __ldg(cp + min(r0 + 1, last));
                    const int32_t i2 = __ldg(cp + min(r0 + 2, last)), i3 = __ldg(cp + min(r0 + 3, last));
                    const uint32_t go = (uint32_t)(lane >> 1) * C::kGroupBytes + (uint32_t)(lane & 1) * 512u;
                    const uint32_t kt = sb + C::oRing + off + go, vt = kt + tile;
#pragma unroll
                    for (int pp = 0; pp < C::P; ++pp)
                        tma_gather4(kt + pp * 1024, &tmK, kfb, h * D + 64 * pp, i0, i1, i2, i3, pol);
#pragma unroll
                    for (int pp = 0; pp < C::P; ++pp)
                        tma_gather4(vt + pp * 1024, &tmV, vfb, h * D + 64 * pp, i0, i1, i2, i3, pol);
                }
                ++seq;
            }
            ++qseq;
        }
        // stop marker
        while (tail <= seq - C::kNS) {
            mbar_wait(bar(B::empty(tail % C::kNS)), (tail / C::kNS) & 1);
            ++tail;
        }
        __syncwarp();
        if (lane == 0) {
            const int s = seq % C::kNS;
            descs[s].rows = -1;
            mbar_arrive(bar(B::kfull(s)));
            mbar_arrive(bar(B::vfull(s)));
        }
        __syncwarp();
    } else if (warp == 1) {
        // ===== MMA issuer ==========================================================================
        constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
        constexpr uint32_t idesc1 = idesc_f16(fmt, 0, 0, 128, 16);  // S^T = K_c . Q_w^T
        constexpr uint32_t idesc2 = idesc_f16(fmt, 1, 0, D, 16);    // O^T = V_c^T . P^T (A MN-major)
        int32_t seq = 0;
        for (;;) {
            const int s = seq % C::kNS;
            const uint32_t ph = (seq / C::kNS) & 1;
            mbar_wait(bar(B::kfull(s)), ph);
            const ChunkDesc dsc = descs[s];
            if (dsc.rows < 0) break;
            const int b = seq & 1;
            if (dsc.flags & 1) mbar_wait(bar(B::qfull(dsc.qslot)), (dsc.flags >> 2) & 1);
            tc_fence_after();
            const uint32_t kt = sb + C::oRing + dsc.ring_off;
            const uint32_t qt = sb + C::oQ + dsc.qslot * C::kQBytes;
            if (lane == 0) {
                if (dsc.rows > 0) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint64_t a = smem_desc_sw128(kt + (kk >> 2) * 1024 + (kk & 3) * 32, 16, C::kGroupBytes);
                        const uint64_t bq = smem_desc_sw128(qt + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
                        mma_f16_ss(tmem + b * 16, a, bq, idesc1, kk > 0 ? 1u : 0u);
                    }
                }
                mma_commit(bar(B::sfull(b)));
                if (dsc.flags & 2) mma_commit(bar(B::qempty(dsc.qslot)));
            }
            __syncwarp();
            mbar_wait(bar(B::pfull(b)), (seq >> 1) & 1);
            mbar_wait(bar(B::vfull(s)), ph);
            tc_fence_after();
            if (lane == 0) {
                if (dsc.rows > 0) {
                    const uint32_t vt = kt + (uint32_t)(dsc.ralloc / 8) * C::kGroupBytes;
                    const uint32_t pt = sb + C::oP + b * C::kPBytes;
                    const int nsteps = (dsc.rows + 15) >> 4;
                    for (int st = 0; st < nsteps; ++st) {
                        const uint64_t a = smem_desc_sw128(vt + st * 2 * C::kGroupBytes, 1024, C::kGroupBytes);
                        const uint64_t bp = smem_desc_sw128(pt + (st >> 2) * 2048 + (st & 3) * 32, 16, 1024);
                        mma_f16_ss(tmem + 32 + b * 16, a, bp, idesc2, st > 0 ? 1u : 0u);
                    }
                }
                mma_commit(bar(B::ofull(b)));
                mma_commit(bar(B::empty(s)));
            }
            __syncwarp();
            ++seq;
        }
    } else {
        // ===== softmax / correction / epilogue (warps 2..5) =======================================
        const int q = warp & 3;          // TMEM lane quadrant this warp may access
        const int p = 32 * q + lane;     // compacted column of the chunk (S^T lane)
        const uint32_t tl = (uint32_t)(32 * q) << 16;
        float* red = reinterpret_cast<float*>(smem + C::oRed);
        float* lred = reinterpret_cast<float*>(smem + C::oLred);
        float m[16], l[16], oacc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) { m[i] = -INFINITY; l[i] = 0.f; oacc[i] = 0.f; }
        int32_t seq = 0;
        for (;;) {
            const int s = seq % C::kNS;
            mbar_wait(bar(B::kfull(s)), (seq / C::kNS) & 1);
            const ChunkDesc dsc = descs[s];
            if (dsc.rows < 0) break;
            if (dsc.flags & 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) { m[i] = -INFINITY; l[i] = 0.f; oacc[i] = 0.f; }
            }
            const uint32_t mask = p < dsc.rows ? (uint32_t)__ldg(masks + dsc.col_base + p) : 0u;
            const int b = seq & 1;
            mbar_wait(bar(B::sfull(b)), (seq >> 1) & 1);
            tc_fence_after();
            float x[16];
            tmem_ld_32x32b_x16(tmem + tl + b * 16, x);
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = ((mask >> i) & 1u) ? x[i] * scale_log2 : -INFINITY;  // Alg.1 l.14
            // chunk row max (Alg.1 l.16)
            const float rm = rowreduce16(x, lane, OpMax());
            if (!(lane & 1)) red[(b * 4 + q) * 16 + ((lane >> 1) & 15)] = rm;
            named_bar_sync(1, 128);
            float alpha[16];
            const float4* r4 = reinterpret_cast<const float4*>(red + b * 64);
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float4 w0 = r4[g], w1 = r4[4 + g], w2 = r4[8 + g], w3 = r4[12 + g];
                const float c0 = fmaxf(fmaxf(w0.x, w1.x), fmaxf(w2.x, w3.x));
                const float c1 = fmaxf(fmaxf(w0.y, w1.y), fmaxf(w2.y, w3.y));
                const float c2 = fmaxf(fmaxf(w0.z, w1.z), fmaxf(w2.z, w3.z));
                const float c3 = fmaxf(fmaxf(w0.w, w1.w), fmaxf(w2.w, w3.w));
                const float cm[4] = {c0, c1, c2, c3};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = 4 * g + e;
                    const float mn = fmaxf(m[i], cm[e]);
                    alpha[i] = mn == -INFINITY ? 1.f : ex2(m[i] - mn);  // e^{m_o - m_i}, 1 if still empty
                    m[i] = mn;
                }
            }
            // E_i = e^{S_i - m_i} (l.17), l_o update (l.18), E -> input dtype in SMEM (l.19)
            uint8_t* pt = smem + C::oP + b * C::kPBytes + (p >> 6) * 2048;
            const uint32_t cchunk = (uint32_t)(p & 63) >> 3, cin = (uint32_t)(p & 7) * 2;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float pv = ((mask >> i) & 1u) ? ex2(x[i] - m[i]) : 0.f;
                l[i] = l[i] * alpha[i] + pv;
                *reinterpret_cast<uint16_t*>(pt + i * 128 + ((cchunk ^ (uint32_t)(i & 7)) << 4) + cin) = to_bits<T>(pv);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(bar(B::pfull(b)));
            // O_i = diag(alpha) O_i + E_i V_j (l.21-22): the chunk's O^T arrives in TMEM
            mbar_wait(bar(B::ofull(b)), (seq >> 1) & 1);
            tc_fence_after();
            if (dsc.rows > 0) {
                float ov[16];
                tmem_ld_32x32b_x16(tmem + tl + 32 + b * 16, ov);
#pragma unroll
                for (int i = 0; i < 16; ++i) oacc[i] = oacc[i] * alpha[i] + ov[i];
            }
            tc_fence_before();
            if (dsc.flags & 2) {
                // l_o = sum over the 128 column partials; O_i = diag(l_o)^-1 O_i (l.24)
                const float rl = rowreduce16(l, lane, OpAdd());
                if (!(lane & 1)) lred[q * 16 + ((lane >> 1) & 15)] = rl;
                named_bar_sync(2, 128);
                const bool has = D == 128 || lane < 16;
                const int f = D == 128 ? p : 16 * q + lane;  // O^T lane -> feature (M = 64 layout)
                if (has) {
                    const int64_t ld = (int64_t)H * D;
                    float* out = O + (int64_t)16 * dsc.rw * ld + (int64_t)dsc.head * D + f;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        if (16 * dsc.rw + i < n_rows) {
                            const float lt = (lred[i] + lred[16 + i]) + (lred[32 + i] + lred[48 + i]);
                            out[(int64_t)i * ld] = lt > 0.f ? oacc[i] * (1.f / lt) : 0.f;
                        }
                    }
                }
            }
            ++seq;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<64>(tmem);
    }
}

// ---- host side ------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

f3s_status make_map(CUtensorMap* map, const void* base, f3s_dtype dtype, int64_t inner, int64_t rows, uint32_t box_rows) {
    EncodeTiledFn enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return F3S_ERR_CUDA; }
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dtype == F3S_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                     const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
        return F3S_ERR_CUDA;
    }
    return F3S_OK;
}

std::atomic<uint32_t> g_call{0};

template <int D, typename T>
f3s_status launch(const AttnArgs& a) {
    using C = Cfg<D>;
    const Plan& p = *a.plan;
    const int64_t out_bytes = (int64_t)p.n_rows * a.heads * D * 4;
    if (p.nnz == 0 || p.n_cols == 0) {  // every row is empty: O = 0 (reading c4)
        F3S_CUDA_TRY(cudaMemsetAsync(a.O, 0, (size_t)out_bytes, a.stream));
        return F3S_OK;
    }
    CUtensorMap mq, mk, mv;
    f3s_status st;
    if ((st = make_map(&mq, a.Q, a.dtype, (int64_t)a.heads * D, p.n_rows, 16)) != F3S_OK) return st;
    if ((st = make_map(&mk, a.K, a.dtype, (int64_t)a.heads * D, p.n_cols, 1)) != F3S_OK) return st;
    if ((st = make_map(&mv, a.V, a.dtype, (int64_t)a.heads * D, p.n_cols, 1)) != F3S_OK) return st;

    static int num_sms[64] = {0};
    const int dev = p.device;
    if (dev < 64 && num_sms[dev] == 0) {
        int v = 0;
        F3S_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        num_sms[dev] = v;
    }
    const int sms = dev < 64 ? num_sms[dev] : 148;
    static std::once_flag attr_once;
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        attr_err = cudaFuncSetAttribute(k_f3s_sm100<D, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    });
    F3S_CUDA_TRY(attr_err);
    const int32_t n_items = (int32_t)((int64_t)p.num_rw * a.heads);
    const int grid = (int)std::min<int64_t>(n_items, (int64_t)sms * C::kCtasPerSm);
    int32_t* counter = p.counters + (g_call.fetch_add(1) % kNumCounterSlots);
    F3S_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int32_t), a.stream));
    k_f3s_sm100<D, T><<<grid, C::kThreads, C::kSmemBytes, a.stream>>>(
        mq, mk, mv, p.rw_ptr, p.cols, p.masks, a.lpt ? p.rw_order : p.rw_natural, counter, n_items, a.heads,
        p.n_rows, a.O, a.scale * 1.4426950408889634f);
    count_launch();
    F3S_CUDA_TRY(cudaGetLastError());
    return F3S_OK;
}

}  // namespace

f3s_status launch_attention_sm100(const AttnArgs& a) {
    if (a.dtype == F3S_FP16) return a.d == 64 ? launch<64, __half>(a) : launch<128, __half>(a);
    return a.d == 64 ? launch<64, __nv_bfloat16>(a) : launch<128, __nv_bfloat16>(a);
}

}  // namespace f3s
