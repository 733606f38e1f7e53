// backward_sm100.cu — the backward of the fused 3S pass on tcgen05 tensor cores (
// "the backward pass ... involves SpMM and SDDMM operations in reverse order").
//
// For O = softmax_row(scale * (Q K^T) (.) A) V and dO = dL/dO (f3s.h f3s_attention_backward):
//   p_ij = 2^(s_ij - LSE_i)   (s in log2 units incl. scale; LSE_i from the forward's (m, l)),
//   D_i  = dO_i . O_i,   dp_ij = dO_i . v_j,   ds_ij = p_ij (dp_ij - D_i),
//   dQ_i = scale sum_j ds_ij k_j,   dK_j = scale sum_i ds_ij q_i,   dV_j = sum_i p_ij dO_i.
// Steps (host, launch_attention_backward_tc):
//   1. the forward in partial mode (unnormalised O, (m, l) per row) and a prep kernel: LSE, D and a
//      copy of dO in the input dtype (the tensor cores multiply 16-bit operands);
//   2. ROW pass over the plan of A, one item per (row window, head), chunks of <= 128 compacted
//      columns (the forward's pipeline with the roles kept): gathered K_c, V_c; per item Q_w, dO_w;
//        MMA1   S^T  = K_c Q_w^T,  dP^T = V_c dO_w^T          (SDDMM twice)
//        elementwise  dS^T = P^T (.) (dP^T - D)               (masked by the bitmap)
//        MMA2   dQ^T += K_c^T dS^T                            (SpMM, accumulated in TMEM)
//   3. COLUMN pass over the plan of A^T (row windows of 16 key columns, compacted query rows):
//      gathered Q_c, dO_c (+ their LSE, D); per item K_w, V_w;
//        MMA1   S = Q_c K_w^T,  dP = dO_c V_w^T;   elementwise P, dS = P (.) (dP - D)
//        MMA2   dV^T += dO_c^T P,   dK^T += Q_c^T dS          (accumulated in TMEM)
// Both passes are deterministic (fixed chunk order per item, no atomics on the data).
//
// One CTA per SM, warps with fixed roles (the forward's structure, attention_sm100.cu):
//   0 index (work queue in LPT order, chunk slots, per-item tiles), 1 MMA1, 2 MMA2, loaders
//   (16-byte cp.async gathers into 128B-swizzled tile slots), two elementwise warpgroups on
//   alternate chunks, one epilogue warpgroup (TMEM accumulators -> shared tile -> TMA store).
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

// PASS 0: rows (dQ), 1: columns (dK, dV).  HG = 4 (head groups, d = 64, every window <= 32
// columns, as in the forward): a chunk holds the window's columns for 4 heads (tile rows 32g.. =
// head g), elementwise warp q works on head q, one epilogue tile covers the 4 heads.
template <int D, int PASS, int HG = 1>
struct BCfg {
    static_assert(HG == 1 || (HG == 4 && D == 64), "head groups: d = 64 only");
    static constexpr int RB = D * 2;                 // bytes of one gathered row of one head
    static constexpr int P = RB / 128;               // 128-byte panels per row
    static constexpr int kRowPitch = 128 * P;
    static constexpr int kGroupBytes = 1024 * P;     // 8 rows (one swizzle atom per panel)
    static constexpr int kMaxRows = 128;
    static constexpr int kTile = (kMaxRows / 8) * kGroupBytes;
    // S/dP TMEM buffers and P/dS shared tiles, chunk slots, per-item tile slots (X and Y: 16 x D
    // each): fewer at d = 128 so that two 32 KB tile slots per gathered operand still fit
    static constexpr int kSB = (D == 128 || HG == 4) ? 2 : 4;
    // (d = 128 columns: 10 slots leave room for a fifth gathered tile, the third Q_c slot)
    static constexpr int kNS = D == 128 ? (PASS == 1 ? 10 : 12) : HG == 4 ? 8 : 16;
    // epilogue warpgroups: head groups (one chunk per item, 4 heads of fp32 gradients per item) use
    // two on alternate items (accumulator buffer e), each with its own staging tiles
    static constexpr int kEpiWGs = HG == 4 ? 2 : 1;
    // per-item X/Y tile slots: the next items' tiles are in flight while one item runs (their TMA
    // latency is exposed with 2 slots and one-chunk items); d = 128 columns: 3 keep five tile slots
    static constexpr int kNQ = HG == 4 ? 2 : (D == 128 && PASS == 1) ? 3 : 4;
    static constexpr int kXBytes = 16 * kRowPitch * HG;  // HG head tiles of 16 x D
    static constexpr int kQBytes = 2 * kXBytes;
    static constexpr int kNT = PASS == 0 ? 1 : 2;    // 16-bit tiles written per chunk: dS (rows); P, dS (cols)
    static constexpr int kPBytes = 16 * kMaxRows * 2;
    static constexpr int kNG = PASS == 0 ? 1 : 2;    // gradient accumulators: dQ; dV, dK
    static constexpr int kOBytes = 16 * D * 4 * HG;  // one [16 x HG*D] fp32 staging tile
    // (LSE, D) pairs per chunk slot: rows, the window's 16 per head; columns none (the elementwise
    // warps load the gathered rows' pairs themselves, off the loaders' cp.async path)
    static constexpr int kScal = PASS == 0 ? 16 * HG : 0;
    static constexpr int kSlotBytes = 32 + kMaxRows * 4 + kMaxRows * 2 + kScal * 8;
    static constexpr int kNumBars = 5 * kNS + 2 * kNQ + 4 * kSB + 4 + 2 * 16;
    static constexpr int kFixed = kNQ * kQBytes + kSB * kNT * kPBytes + kEpiWGs * kNG * kOBytes + kNS * kSlotBytes +
                                  kNumBars * 8 + 64 + 16;
    // gathered tile slots: both operands live until MMA2 in the column pass; in the row pass V_c is
    // free after MMA1, so K_c (read by MMA1 and MMA2) gets the remaining slots
    static constexpr int kSlotsAll = (227 * 1024 - kFixed) / kTile;
    // (the loaders issue a chunk's A1 rows before they wait for its A2 slot, so an odd slot goes to A1)
    static constexpr int kN2 = PASS == 0 ? 2 : kSlotsAll / 2;
    static constexpr int kN1 = PASS == 0 ? (kSlotsAll - 2 < 16 ? kSlotsAll - 2 : 16) : kSlotsAll - kSlotsAll / 2;
    static_assert(kN1 >= 2 && kN2 >= 2 && kN1 <= 16 && kN2 <= 16, "tile slots per operand");
    static constexpr int oT1 = 0, oT2 = kN1 * kTile;
    static constexpr int oQ = (kN1 + kN2) * kTile;
    static constexpr int oP = oQ + kNQ * kQBytes;
    static constexpr int oOst = oP + kSB * kNT * kPBytes;
    static constexpr int oSlot = oOst + kEpiWGs * kNG * kOBytes;
    static constexpr int oRec = oSlot + kNS * kSlotBytes;  // int4 [2] accumulator records
    static constexpr int oBar = oRec + 64;
    static constexpr int oTmem = oBar + kNumBars * 8;
    static constexpr int kSmemBytes = oTmem + 16;
    static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");
    // TMEM: S (kSB x HG x 16), dP (kSB x HG x 16), gradient accumulators (2 item buffers x HG x kNG x 16)
    static constexpr int kTmS = 0, kTmP = 16 * kSB * HG, kTmG = 32 * kSB * HG;
    static constexpr int kTmUsed = kTmG + 2 * HG * kNG * 16;
    static constexpr int kTmemCols = kTmUsed <= 256 ? 256 : 512;
    static_assert(kTmUsed <= 512, "TMEM columns");
    static constexpr int kLoaderWarps = D == 128 ? 8 : 6;
    static constexpr int kLoader0 = 3, kEw0 = kLoader0 + kLoaderWarps, kEpi0 = kEw0 + 8;
    static constexpr int kTileWarp = kEpi0 + 4 * kEpiWGs;  // per-item X/Y tiles (TMA)
    static constexpr int kThreads = 32 * (kTileWarp + 1);
    static constexpr int kBatch = 8;
};

template <int D, int PASS, int HG> struct BBars {
    using C = BCfg<D, PASS, HG>;
    __host__ __device__ static constexpr int idxfull(int s) { return s; }
    __host__ __device__ static constexpr int a1full(int s) { return C::kNS + s; }
    __host__ __device__ static constexpr int a2full(int s) { return 2 * C::kNS + s; }
    __host__ __device__ static constexpr int empty(int s) { return 3 * C::kNS + s; }
    __host__ __device__ static constexpr int xyfull(int q) { return 5 * C::kNS + q; }
    __host__ __device__ static constexpr int xyempty(int q) { return 5 * C::kNS + C::kNQ + q; }
    static constexpr int kB0 = 5 * C::kNS + 2 * C::kNQ;
    __host__ __device__ static constexpr int sfull(int b) { return kB0 + b; }
    __host__ __device__ static constexpr int sfree(int b) { return kB0 + C::kSB + b; }
    __host__ __device__ static constexpr int pfull(int b) { return kB0 + 2 * C::kSB + b; }
    __host__ __device__ static constexpr int pempty(int b) { return kB0 + 3 * C::kSB + b; }
    __host__ __device__ static constexpr int gfull(int a) { return kB0 + 4 * C::kSB + a; }
    __host__ __device__ static constexpr int gempty(int a) { return kB0 + 4 * C::kSB + 2 + a; }
    __host__ __device__ static constexpr int t1free(int t) { return kB0 + 4 * C::kSB + 4 + t; }
    __host__ __device__ static constexpr int t2free(int t) { return kB0 + 4 * C::kSB + 4 + 16 + t; }
};

template <int kScal> struct __align__(16) BSlot {
    int32_t rw, head, rows, qslot, flags, pad0, pad1, pad2;
    int32_t cols[128];
    uint16_t masks[128];
    float2 ld[kScal];  // (LSE in log2 units, D = dO . O) of the window's 16 query rows per head (rows pass)
};
template <> struct __align__(16) BSlot<0> {
    int32_t rw, head, rows, qslot, flags, pad0, pad1, pad2;
    int32_t cols[128];
    uint16_t masks[128];
};

template <typename T> __device__ __forceinline__ uint32_t bpack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t bpack2<__half>(float lo, float hi) { return pack_f16x2(lo, hi); }
template <> __device__ __forceinline__ uint32_t bpack2<__nv_bfloat16>(float lo, float hi) { return pack_bf16x2(lo, hi); }

// store 16 values of chunk entry p as row p of an MN-major SW32 [128 x 16] B-operand tile (the
// forward's P^T layout): one 32-byte row per entry, 8 rows per 256-byte atom, halves swapped when
// bit 2 of p is set
template <typename T>
__device__ __forceinline__ void store_tile_row(uint8_t* tile, int p, const float (&v)[16]) {
    uint4* prow = reinterpret_cast<uint4*>(tile + (p >> 3) * 256 + (p & 7) * 32);
    const int sw = (p >> 2) & 1;
    prow[sw] = make_uint4(bpack2<T>(v[0], v[1]), bpack2<T>(v[2], v[3]), bpack2<T>(v[4], v[5]), bpack2<T>(v[6], v[7]));
    prow[sw ^ 1] = make_uint4(bpack2<T>(v[8], v[9]), bpack2<T>(v[10], v[11]), bpack2<T>(v[12], v[13]),
                              bpack2<T>(v[14], v[15]));
}

template <int D, typename T, int PASS, int HG>
__global__ void __launch_bounds__(BCfg<D, PASS, HG>::kThreads, 1)
k_bwd_sm100(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
            const __grid_constant__ CUtensorMap tmG1, const __grid_constant__ CUtensorMap tmG2,
            const int4* __restrict__ meta, const int32_t* __restrict__ kcols, const uint16_t* __restrict__ kmasks,
            int32_t* __restrict__ counter, int32_t n_items, int32_t heavy_items, int32_t H,
            const uint8_t* __restrict__ A1g, const uint8_t* __restrict__ A2g, int64_t ld_bytes,
            const float2* __restrict__ ld_t, int64_t nq16, float scale_log2,
            float g2scale, float g1scale, int32_t out16) {
    using C = BCfg<D, PASS, HG>;
    using B = BBars<D, PASS, HG>;
    using Slot = BSlot<C::kScal>;
    static_assert(sizeof(Slot) == C::kSlotBytes, "slot layout");
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = smem_u32(smem);
    if (sb & 1023) __trap();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto bar = [&](int i) -> uint32_t { return sb + C::oBar + 8u * i; };
    Slot* slots = reinterpret_cast<Slot*>(smem + C::oSlot);
    int4* rec = reinterpret_cast<int4*>(smem + C::oRec);

    for (int i = threadIdx.x; i < (C::kN1 + C::kN2) * C::kTile / 16; i += blockDim.x)
        reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < C::kNS * C::kSlotBytes / 16; i += blockDim.x)
        reinterpret_cast<int4*>(smem + C::oSlot)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kNS; ++s) {
            mbar_init(bar(B::idxfull(s)), 1);
            mbar_init(bar(B::a1full(s)), 32 * C::kLoaderWarps);
            mbar_init(bar(B::a2full(s)), 32 * C::kLoaderWarps);
            mbar_init(bar(B::empty(s)), 1);
        }
        for (int q = 0; q < C::kNQ; ++q) {
            mbar_init(bar(B::xyfull(q)), 1);
            mbar_init(bar(B::xyempty(q)), 1);
        }
        for (int b = 0; b < C::kSB; ++b) {
            mbar_init(bar(B::sfull(b)), 1);
            mbar_init(bar(B::sfree(b)), 4);
            mbar_init(bar(B::pfull(b)), 128);
            mbar_init(bar(B::pempty(b)), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar(B::gfull(a)), 2);  // MMA completion + the MMA2 warp's record
            mbar_init(bar(B::gempty(a)), 128);
        }
        for (int t = 0; t < C::kN1; ++t) mbar_init(bar(B::t1free(t)), 1);
        for (int t = 0; t < C::kN2; ++t) mbar_init(bar(B::t2free(t)), 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmY);
        tma_prefetch_desc(&tmG1);
        if (PASS == 1) tma_prefetch_desc(&tmG2);
    }
    if (warp == 1) {
        tmem_alloc<C::kTmemCols>(sb + C::oTmem);
        tmem_relinquish();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::oTmem);
    constexpr int chunk_rows = C::kMaxRows;

    if (warp == 0) {
        // ===== index warp: items in LPT order (heavy prefix one per claim) -> chunk slots =====
        int32_t seq = 0, qseq = 0, last = 0;
        bool done = false;
        const int batch = max(1, min(C::kBatch, n_items / (4 * (int)gridDim.x)));  // as the forward's
        while (!done) {
            const int nclaim = last < heavy_items ? 1 : batch;
            int32_t it = 0x7FFFFFFF;
            int4 mt = make_int4(0, 0, 0, 0);
            if (lane < nclaim) {
                it = atomicAdd(counter, 1);
                if (it < n_items) mt = __ldg(meta + it / (H / HG));
            }
            __syncwarp();
            last = __shfl_sync(0xffffffffu, it, nclaim - 1);
            for (int b = 0; b < nclaim; ++b) {
                const int32_t itb = __shfl_sync(0xffffffffu, it, b);
                const int32_t k = __shfl_sync(0xffffffffu, mt.x, b);
                const int32_t cb8 = __shfl_sync(0xffffffffu, mt.y, b);
                const int32_t w = __shfl_sync(0xffffffffu, mt.z, b);
                if (itb >= n_items) { done = true; continue; }
                const int32_t h = (itb - (itb / (H / HG)) * (H / HG)) * HG;  // (first) head
                const int nch = w > 0 ? (w + chunk_rows - 1) / chunk_rows : 1;
                const int qs = qseq % C::kNQ;  // the item's X/Y slot (loaded by the tile warp)
                const int qph = (qseq / C::kNQ) & 1;
                for (int j = 0; j < nch; ++j) {
                    const int rows = w > 0 ? min(chunk_rows, w - chunk_rows * j) : 0;
                    const int s = seq % C::kNS;
                    if (lane == 0) {
                        mbar_wait(bar(B::empty(s)), ((seq / C::kNS) & 1) ^ 1);
                        Slot& sl = slots[s];
                        sl.rw = k;
                        sl.head = h;
                        sl.rows = rows;
                        sl.qslot = qs;
                        sl.flags = (j == 0 ? 1 : 0) | (j == nch - 1 ? 2 : 0) | (qph << 2);
                        const uint32_t fb = bar(B::idxfull(s));
                        const uint32_t r8 = (uint32_t)((rows + 7) & ~7);
                        const uint32_t scal = PASS == 0 ? 128u * HG : 0u;  // rows: the window's 16 (LSE, D) per head
                        mbar_arrive_expect_tx(fb, (rows > 0 ? r8 * 6u : 0u) + scal);
                        if (rows > 0) {
                            bulk_g2s(smem_u32(sl.cols), kcols + cb8 + chunk_rows * j, r8 * 4u, fb);
                            bulk_g2s(smem_u32(sl.masks), kmasks + cb8 + chunk_rows * j, r8 * 2u, fb);
                        }
                        if constexpr (PASS == 0) {
#pragma unroll
                            for (int g = 0; g < HG; ++g)
                                bulk_g2s(smem_u32(sl.ld + 16 * g), ld_t + (h + g) * nq16 + 16 * (int64_t)k, 128u, fb);
                        }
                    }
                    ++seq;
                }
                ++qseq;
            }
        }
        if (lane == 0) {
            for (int w = 0; w < 2; ++w, ++seq) {  // one stop marker per elementwise warpgroup
                const int s = seq % C::kNS;
                mbar_wait(bar(B::empty(s)), ((seq / C::kNS) & 1) ^ 1);
                slots[s].rows = -1 - w;
                mbar_arrive(bar(B::idxfull(s)));
            }
        }
        __syncwarp();
    } else if (warp == C::kTileWarp) {
        // ===== tile warp: the item's 16-row tiles X and Y (rows: Q_w, dO_w; cols: K_w, V_w) =======
        // walks the chunk slots in order and loads at each item's first chunk, so that waiting for
        // a free X/Y slot never holds the index warp back from filling chunk slots ahead
        if (lane == 0) {
            for (int32_t seq = 0;; ++seq) {
                const int s = seq % C::kNS;
                mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);
                const Slot& sl = slots[s];
                const int rows = sl.rows, flags = sl.flags;
                if (rows < 0) break;
                if (!(flags & 1)) continue;
                const int qs = sl.qslot, qph = (flags >> 2) & 1, k = sl.rw, h = sl.head;
                mbar_wait(bar(B::xyempty(qs)), qph ^ 1);
                mbar_arrive_expect_tx(bar(B::xyfull(qs)), C::kQBytes);
                const uint32_t xd = sb + C::oQ + qs * C::kQBytes;
#pragma unroll
                for (int g = 0; g < HG; ++g)
#pragma unroll
                    for (int pp = 0; pp < C::P; ++pp) {
                        const uint32_t o = g * 16 * C::kRowPitch + pp * 2048;
                        tma_load_2d(xd + o, &tmX, bar(B::xyfull(qs)), (h + g) * D + 64 * pp, 16 * k);
                        tma_load_2d(xd + C::kXBytes + o, &tmY, bar(B::xyfull(qs)), (h + g) * D + 64 * pp, 16 * k);
                    }
            }
        }
        __syncwarp();
    } else if (warp >= C::kLoader0 && warp < C::kLoader0 + C::kLoaderWarps) {
        // ===== loaders: the chunk's A1 and A2 rows ===============================================
        constexpr int kPieces = C::RB / 16;
        constexpr int kRowsPerOp = 32 / kPieces;
        constexpr int kIters = (C::kMaxRows / kRowsPerOp + C::kLoaderWarps - 1) / C::kLoaderWarps;
        const int lw = warp - C::kLoader0;
        const int piece = lane % kPieces, rsub = lane / kPieces;
        const int pnl = piece >> 3, cc = piece & 7;
        for (int32_t seq = 0;; ++seq) {
            const int s = seq % C::kNS;
            mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);
            Slot& sl = slots[s];
            const int rows = sl.rows;
            const uint32_t f1 = bar(B::a1full(s)), f2 = bar(B::a2full(s));
            if (rows < 0) {
                mbar_arrive(f1);
                mbar_arrive(f2);
                break;
            }
            const int h = sl.head;
            const int t1 = seq % C::kN1, t2 = seq % C::kN2;
            const uint32_t d1 = sb + C::oT1 + t1 * C::kTile + pnl * 1024;
            const uint32_t d2 = sb + C::oT2 + t2 * C::kTile + pnl * 1024;
            const uint8_t* b1 = A1g + (int64_t)h * C::RB + piece * 16;
            const uint8_t* b2 = A2g + (int64_t)h * C::RB + piece * 16;
            // HG = 1: tile row r = compacted column r.  HG = 4: tile row 32g + r = column r of head h + g
            const int ops = HG == 1 ? (rows + kRowsPerOp - 1) / kRowsPerOp : C::kMaxRows / kRowsPerOp;
            mbar_wait(bar(B::t1free(t1)), ((seq / C::kN1) & 1) ^ 1);
            int64_t jj[kIters];
            uint32_t dst[kIters];
            int rr[kIters];
            bool ok[kIters];
#pragma unroll
            for (int i = 0; i < kIters; ++i) {
                const int t = lw + i * C::kLoaderWarps;
                const int tr = t * kRowsPerOp + rsub;  // tile row
                const int r = HG == 1 ? tr : (tr & 31);
                ok[i] = t < ops && r < rows;
                rr[i] = tr;
                jj[i] = ok[i] ? sl.cols[r] : 0;
                dst[i] = (uint32_t)(tr >> 3) * C::kGroupBytes + (uint32_t)(tr & 7) * 128 + (uint32_t)((cc ^ (tr & 7)) << 4);
            }
#pragma unroll
            for (int i = 0; i < kIters; ++i)
                if (ok[i]) cp_async_16(d1 + dst[i], b1 + jj[i] * ld_bytes + (HG == 1 ? 0 : (int64_t)(rr[i] >> 5) * C::RB));
            cp_async_mbar_arrive(f1);
            // the A2 slot is awaited only now: with more A1 than A2 slots the A1 rows of the next
            // chunk are already on their way while the A2 slot drains
            mbar_wait(bar(B::t2free(t2)), ((seq / C::kN2) & 1) ^ 1);
#pragma unroll
            for (int i = 0; i < kIters; ++i)
                if (ok[i]) cp_async_16(d2 + dst[i], b2 + jj[i] * ld_bytes + (HG == 1 ? 0 : (int64_t)(rr[i] >> 5) * C::RB));
            cp_async_mbar_arrive(f2);
        }
    } else if (warp == 1) {
        // ===== MMA1: S^T = A1_c . X^T and dP^T = A2_c . Y^T (swap-AB, M = 128, N = 16) =========
        constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
        constexpr uint32_t idesc1 = idesc_f16(fmt, 0, 0, 128, 16 * HG);
        const uint64_t dA = smem_desc_sw128(0, 16, C::kGroupBytes);
        const uint64_t dX = smem_desc_sw128(0, 16, 1024);
        for (int32_t n1 = 0;; ++n1) {
            const int s = n1 % C::kNS, b = n1 % C::kSB;
            mbar_wait(bar(B::a1full(s)), (n1 / C::kNS) & 1);
            const Slot& sl = slots[s];
            const int rows = sl.rows, flags = sl.flags, qslot = sl.qslot;
            if (rows < 0) break;
            mbar_wait(bar(B::sfree(b)), ((n1 / C::kSB) & 1) ^ 1);
            if (flags & 1) mbar_wait(bar(B::xyfull(qslot)), (flags >> 2) & 1);
            tc_fence_after();
            // S^T from A1 as soon as A1 has landed, then dP^T once A2 has (the loaders issue A1 first)
            const uint64_t a1 = dA + ((sb + C::oT1 + (n1 % C::kN1) * C::kTile) >> 4);
            const uint64_t a2 = dA + ((sb + C::oT2 + (n1 % C::kN2) * C::kTile) >> 4);
            const uint64_t bx = dX + ((sb + C::oQ + qslot * C::kQBytes) >> 4);
            const uint64_t by = dX + ((sb + C::oQ + qslot * C::kQBytes + C::kXBytes) >> 4);
            // HG > 1: the HG head tiles of X (Y) form one [16 HG x 64] K-major tile: one N = 16 HG MMA
            // per K-step; head g's tile rows (lanes 32g ..) are read back from columns 16g .. only
            if (rows > 0) {
#pragma unroll
                for (int kk = 0; kk < C::RB / 32; ++kk) {
                    const uint32_t ko = ((kk >> 2) * 1024 + (kk & 3) * 32) >> 4;
                    const uint32_t bo = ((kk >> 2) * 2048 + (kk & 3) * 32) >> 4;
                    mma_f16_ss_warp(tmem + C::kTmS + b * HG * 16, a1 + ko, bx + bo, idesc1, kk > 0 ? 1u : 0u);
                }
            }
            mbar_wait(bar(B::a2full(s)), (n1 / C::kNS) & 1);
            tc_fence_after();
            if (rows > 0) {
#pragma unroll
                for (int kk = 0; kk < C::RB / 32; ++kk) {
                    const uint32_t ko = ((kk >> 2) * 1024 + (kk & 3) * 32) >> 4;
                    const uint32_t bo = ((kk >> 2) * 2048 + (kk & 3) * 32) >> 4;
                    mma_f16_ss_warp(tmem + C::kTmP + b * HG * 16, a2 + ko, by + bo, idesc1, kk > 0 ? 1u : 0u);
                }
            }
            mma_commit_warp(bar(B::sfull(b)));
            if (PASS == 0) mma_commit_warp(bar(B::t2free(n1 % C::kN2)));  // rows: V_c is MMA1's alone
            if (flags & 2) mma_commit_warp(bar(B::xyempty(qslot)));
        }
        __syncwarp();
    } else if (warp == 2) {
        // ===== MMA2: gradients accumulated in TMEM over the item's chunks ==========================
        //   rows: dQ^T += K_c^T dS^T;   cols: dV^T += dO_c^T P,  dK^T += Q_c^T dS
        constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
        constexpr uint32_t idesc2 = idesc_f16(fmt, 1, 1, D, 16);
        const uint64_t dA = smem_desc_sw128(0, 1024, C::kGroupBytes);
        const uint64_t dPt = smem_desc_sw32(0, 4096, 256);
        int32_t item = 0;
        bool any = false;
        for (int32_t n2 = 0;; ++n2) {
            const int s = n2 % C::kNS, b = n2 % C::kSB, a = item & 1;
            mbar_wait(bar(B::a1full(s)), (n2 / C::kNS) & 1);
            if (PASS == 1) mbar_wait(bar(B::a2full(s)), (n2 / C::kNS) & 1);
            const Slot& sl = slots[s];
            const int rows = sl.rows, flags = sl.flags, rw = sl.rw, hd = sl.head;
            if (rows < 0) {  // tell the epilogue warpgroup(s) to stop (their next records)
                for (int e = 0; e < C::kEpiWGs; ++e) {
                    const int it = item + e, ae = it & 1;
                    mbar_wait(bar(B::gempty(ae)), ((it >> 1) & 1) ^ 1);
                    if (lane == 0) {
                        rec[ae] = make_int4(-1, 0, 0, 0);
                        mbar_arrive(bar(B::gfull(ae)));
                        mbar_arrive(bar(B::gfull(ae)));
                    }
                }
                break;
            }
            mbar_wait(bar(B::pfull(b)), (n2 / C::kSB) & 1);
            if (flags & 1) {
                mbar_wait(bar(B::gempty(a)), ((item >> 1) & 1) ^ 1);
                any = false;
            }
            tc_fence_after();
            if (rows > 0) {
                const uint64_t a1 = dA + ((sb + C::oT1 + (n2 % C::kN1) * C::kTile) >> 4);
                const uint64_t a2 = dA + ((sb + C::oT2 + (n2 % C::kN2) * C::kTile) >> 4);
                const uint64_t p0 = dPt + ((sb + C::oP + b * C::kNT * C::kPBytes) >> 4);
                const int nsteps = HG == 1 ? (rows + 15) / 16 : 2;  // head groups: 32 tile rows per head
#pragma unroll
                for (int g = 0; g < HG; ++g) {
                    const uint32_t gacc = C::kTmG + (a * HG + g) * 16 * C::kNG;  // this item buffer's head g
                    for (int st = 0; st < nsteps; ++st) {
                        const uint32_t acc = (any || st > 0) ? 1u : 0u;
                        const uint32_t ao = (g * 4 * C::kGroupBytes + st * 2 * C::kGroupBytes) >> 4;
                        const uint32_t po = (g * 1024 + st * 512) >> 4;
                        if (PASS == 0) {
                            mma_f16_ss_warp(tmem + gacc, a1 + ao, p0 + po, idesc2, acc);
                        } else {
                            mma_f16_ss_warp(tmem + gacc, a2 + ao, p0 + po, idesc2, acc);                         // dV
                            mma_f16_ss_warp(tmem + gacc + 16, a1 + ao, p0 + (C::kPBytes >> 4) + po, idesc2, acc);  // dK
                        }
                    }
                }
                any = true;
            }
            mma_commit_warp(bar(B::pempty(b)));
            mma_commit_warp(bar(B::t1free(n2 % C::kN1)));
            if (PASS == 1) mma_commit_warp(bar(B::t2free(n2 % C::kN2)));
            mma_commit_warp(bar(B::empty(s)));
            if (flags & 2) {
                if (lane == 0) rec[a] = make_int4(rw, hd, any ? 1 : 0, 0);
                mma_commit_warp(bar(B::gfull(a)));
                __syncwarp();
                if (lane == 0) mbar_arrive(bar(B::gfull(a)));
                ++item;
            }
            __syncwarp();
        }
        __syncwarp();
    } else if (warp < C::kEpi0) {
        // ===== elementwise warpgroups (alternate chunks) ==========================================
        // TMEM lane p = chunk entry p (rows: compacted column j; cols: compacted query row i), the 16
        // TMEM columns = the window's 16 query rows (rows) or key columns (cols)
        const int q = warp & 3;
        const int p = 32 * q + lane;  // tile row = TMEM lane
        const int col = HG == 1 ? p : lane;  // compacted column / row of the chunk (HG = 4: of head q)
        const int wg = (warp - C::kEw0) >> 2;
        const uint32_t tl = (uint32_t)(32 * q) << 16;
        const int hb = HG == 1 ? 0 : q;  // the warp's head within the group
        for (int32_t seq = wg;; seq += 2) {
            const int s = seq % C::kNS, b = seq % C::kSB;
            const uint32_t bph = (seq / C::kSB) & 1;
            mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);
            const Slot& sl = slots[s];
            const int rows = sl.rows;
            if (rows < 0) break;
            const uint32_t mask = col < rows ? (uint32_t)sl.masks[col] : 0u;
            float2 ld_p = make_float2(0.f, 0.f);
            if constexpr (PASS == 1) {  // the (LSE, D) of this lane's gathered query row (L2; its
                                        // latency hides behind the gathers and MMA1)
                if (col < rows) ld_p = __ldg(ld_t + (int64_t)(sl.head + hb) * nq16 + sl.cols[col]);
            }
            mbar_wait(bar(B::sfull(b)), bph);
            tc_fence_after();
            float x[16], y[16];
            tmem_ld_32x32b_x16(tmem + tl + C::kTmS + (b * HG + hb) * 16, x);
            tmem_ld_32x32b_x16(tmem + tl + C::kTmP + (b * HG + hb) * 16, y);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(B::sfree(b)));
            float pr[16], ds[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float l = ld_p.x, dd = ld_p.y;
                if constexpr (PASS == 0) {
                    l = sl.ld[16 * hb + i].x;
                    dd = sl.ld[16 * hb + i].y;
                }
                const float pv = ((mask >> i) & 1u) ? ex2(fmaf(x[i], scale_log2, -l)) : 0.f;
                pr[i] = pv;
                ds[i] = pv * (y[i] - dd);
            }
            mbar_wait(bar(B::pempty(b)), bph ^ 1);
            uint8_t* tile = smem + C::oP + b * C::kNT * C::kPBytes;
            if (PASS == 0) {
                store_tile_row<T>(tile, p, ds);
            } else {
                store_tile_row<T>(tile, p, pr);
                store_tile_row<T>(tile + C::kPBytes, p, ds);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(bar(B::pfull(b)));
        }
    } else {
        // ===== epilogue: accumulators -> [16 x D] fp32 tiles -> TMA stores =========================
        const int q = warp & 3;
        const uint32_t tl = (uint32_t)(32 * q) << 16;
        const bool has = D == 128 || lane < 16;
        const int f = D == 128 ? 32 * q + lane : 16 * q + lane;  // accumulator lane -> feature
        const int e = (warp - C::kEpi0) >> 2;  // epilogue warpgroup: items e, e + kEpiWGs, ..
        const bool lead = threadIdx.x == 32 * (C::kEpi0 + 4 * e);
        const uint32_t ost = C::oOst + e * C::kNG * C::kOBytes;
        for (int32_t item = e;; item += C::kEpiWGs) {
            const int a = item & 1;
            mbar_wait(bar(B::gfull(a)), (item >> 1) & 1);
            const int4 r = rec[a];
            if (r.x < 0) break;
            tc_fence_after();
            const bool nz = r.z != 0;  // an item with no entries has an untouched accumulator: zeros
            if (lead) bulk_wait_group_read<0>();
            named_bar_sync(3 + e, 128);
            // staging tiles at ost (G1) and ost + kOBytes (G2): fp32, or the input dtype (out16,
            // f3s_attention_backward_saved_lp: the fp32 accumulators rounded once, RNE)
            float* o1 = reinterpret_cast<float*>(smem + ost);
            float* o2 = reinterpret_cast<float*>(smem + ost + C::kOBytes);
            T* h1 = reinterpret_cast<T*>(o1);
            T* h2 = reinterpret_cast<T*>(o2);
#pragma unroll 1
            for (int g = 0; g < HG; ++g) {  // [16 x HG*D] tiles: head g in columns g*D ..
                float g1[16], g2[16];
                const uint32_t gacc = C::kTmG + (a * HG + g) * 16 * C::kNG;
                tmem_ld_32x32b_x16(tmem + tl + gacc, g1);
                if (PASS == 1) tmem_ld_32x32b_x16(tmem + tl + gacc + 16, g2);
                if (has) {
                    if (out16) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            h1[i * (HG * D) + g * D + f] = T(nz ? g1[i] * g1scale : 0.f);
                            if (PASS == 1) h2[i * (HG * D) + g * D + f] = T(nz ? g2[i] * g2scale : 0.f);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            o1[i * (HG * D) + g * D + f] = nz ? g1[i] * g1scale : 0.f;
                            if (PASS == 1) o2[i * (HG * D) + g * D + f] = nz ? g2[i] * g2scale : 0.f;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(bar(B::gempty(a)));
            fence_proxy_async_smem();
            named_bar_sync(3 + e, 128);
            if (lead) {
                tma_store_2d(&tmG1, sb + ost, r.y * D, 16 * r.x);
                if (PASS == 1) tma_store_2d(&tmG2, sb + ost + C::kOBytes, r.y * D, 16 * r.x);
                bulk_commit_group();
            }
        }
        if (lead) bulk_wait_group<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

// (LSE, D) per row and head -- LSE_i = m_i + log2(l_i) in log2 units incl. scale (+inf for an empty
// row: p = 0), D_i = dO_i . O_i -- and dO in the input dtype, from the forward's partial outputs
// (unnormalised O, (m, l)) or the saved outputs of f3s_attention_fwd (normalized: O / l, (m, l)).
// D / 4 lanes per (row, head), 16-byte loads, kU (row, head) pairs per group in flight; head-major
// output ld_t[h][nq16].  kLp: dO is given in the input dtype (f3s_attention_backward_saved_lp): it is
// read as such and used in place by the passes (no dO16 written).
template <int D, typename T, bool kLp = false>
__global__ void __launch_bounds__(256) k_bwd_prep(const float* __restrict__ Op, const float2* __restrict__ ml,
                                                  const void* __restrict__ dOv, int64_t n_rows, int32_t H,
                                                  int64_t nq16, float2* __restrict__ ld_t, T* __restrict__ dO16,
                                                  int32_t normalized) {
    const float* __restrict__ dO = static_cast<const float*>(dOv);
    const T* __restrict__ dOl = static_cast<const T*>(dOv);
    constexpr int L = D / 4, kU = 4;
    const int sub = threadIdx.x % L;
    const int64_t ng = (int64_t)gridDim.x * (blockDim.x / L);
    const int64_t gid = (int64_t)blockIdx.x * (blockDim.x / L) + threadIdx.x / L;
    const int64_t total = n_rows * H;
    for (int64_t r0 = gid; r0 < total; r0 += ng * kU) {
        float4 o[kU], g[kU];
        float2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t rh = r0 + u * ng;
            if (rh < total) {
                o[u] = __ldg(reinterpret_cast<const float4*>(Op + rh * D) + sub);
                if constexpr (kLp) {
                    const uint2 w = __ldg(reinterpret_cast<const uint2*>(dOl + rh * D) + sub);
                    const T* t = reinterpret_cast<const T*>(&w);
                    g[u] = make_float4((float)t[0], (float)t[1], (float)t[2], (float)t[3]);
                } else {
                    g[u] = __ldg(reinterpret_cast<const float4*>(dO + rh * D) + sub);
                }
                v[u] = __ldg(ml + rh);
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t rh = r0 + u * ng;
            const float inv = normalized ? 1.f : v[u].y > 0.f ? 1.f / v[u].y : 0.f;  // saved O is already O / l
            float acc = fmaf(g[u].x, o[u].x * inv, fmaf(g[u].y, o[u].y * inv, fmaf(g[u].z, o[u].z * inv, g[u].w * (o[u].w * inv))));
#pragma unroll
            for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (rh < total) {
                if constexpr (!kLp) {
                    uint2 pk;
                    if constexpr (std::is_same<T, __half>::value) {
                        pk.x = pack_f16x2(g[u].x, g[u].y);
                        pk.y = pack_f16x2(g[u].z, g[u].w);
                    } else {
                        pk.x = pack_bf16x2(g[u].x, g[u].y);
                        pk.y = pack_bf16x2(g[u].z, g[u].w);
                    }
                    reinterpret_cast<uint2*>(dO16 + rh * D)[sub] = pk;
                }
                if (sub == 0) {
                    const int64_t i = rh / H;
                    const int h = (int)(rh - i * H);
                    ld_t[h * nq16 + i] = make_float2(v[u].y > 0.f ? v[u].x + __log2f(v[u].y) : INFINITY, acc);
                }
            }
        }
    }
}

template <int D, typename T, int PASS, int HG>
f3s_status launch_pass_hg(const Plan& p, const void* X, const void* Y, const void* A1, const void* A2, void* G1,
                          void* G2, bool out16, const float2* ld_t, int64_t nq16, int H, float scale,
                          int sms, cudaStream_t stream) {
    using C = BCfg<D, PASS, HG>;
    if (p.num_rw == 0) return F3S_OK;
    const f3s_dtype dt = std::is_same<T, __half>::value ? F3S_FP16 : F3S_BF16;
    const int64_t ld = (int64_t)H * D;
    CUtensorMap mx, my, mg1, mg2;
    f3s_status st;
    if ((st = make_map(&mx, X, dt, ld, p.n_rows, ld, 16)) != F3S_OK) return st;
    if ((st = make_map(&my, Y, dt, ld, p.n_rows, ld, 16)) != F3S_OK) return st;
    const CUtensorMapDataType gt = !out16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : dt == F3S_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    if ((st = make_map(&mg1, G1, gt, ld, p.n_rows, ld, D * HG, 16, CU_TENSOR_MAP_SWIZZLE_NONE)) != F3S_OK) return st;
    mg2 = mg1;
    if (PASS == 1 && (st = make_map(&mg2, G2, gt, ld, p.n_rows, ld, D * HG, 16, CU_TENSOR_MAP_SWIZZLE_NONE)) != F3S_OK)
        return st;
    static std::atomic<uint64_t> attr_set{0};
    static std::mutex mu;
    if (!(attr_set.load() >> p.device & 1)) {
        std::lock_guard<std::mutex> lock(mu);
        if (!(attr_set.load() >> p.device & 1)) {
            F3S_CUDA_TRY(cudaFuncSetAttribute(k_bwd_sm100<D, T, PASS, HG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              C::kSmemBytes));
            attr_set.fetch_or(uint64_t(1) << p.device);
        }
    }
    const int64_t n_items64 = (int64_t)p.num_rw * (H / HG);
    if (n_items64 > 0x7FFFFFFF) { set_error("too many work items"); return F3S_ERR_UNSUPPORTED; }
    char* scratch = nullptr;
    F3S_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&scratch), 256, stream));
    cudaError_t err = cudaMemsetAsync(scratch, 0, sizeof(int32_t), stream);
    if (err == cudaSuccess) {
        const int grid = (int)std::min<int64_t>(n_items64, sms);
        k_bwd_sm100<D, T, PASS, HG><<<grid, C::kThreads, C::kSmemBytes, stream>>>(
            mx, my, mg1, mg2, p.meta_lpt, p.kcols, p.kmasks, reinterpret_cast<int32_t*>(scratch), (int32_t)n_items64,
            (int32_t)std::min<int64_t>((int64_t)p.n_heavy_lpt * (H / HG), 0x7FFFFFFF), H,
            static_cast<const uint8_t*>(A1), static_cast<const uint8_t*>(A2), ld * 2, ld_t, nq16,
            scale * 1.4426950408889634f, scale, PASS == 0 ? scale : 1.f, out16 ? 1 : 0);
        count_launch();
        err = cudaGetLastError();
    }
    const cudaError_t ferr = scratch_free(scratch, stream);
    F3S_CUDA_TRY(err);
    F3S_CUDA_TRY(ferr);
    return F3S_OK;
}

// head groups of 4 when d = 64, H % 4 == 0 and every window of the pass's plan has <= 32 columns
template <int D, typename T, int PASS>
f3s_status launch_pass(const Plan& p, const void* X, const void* Y, const void* A1, const void* A2, void* G1,
                       void* G2, bool out16, const float2* ld_t, int64_t nq16, int H, float scale,
                       int sms, cudaStream_t stream) {
    if constexpr (D == 64) {
        if (H % 4 == 0 && p.max_width <= 32)
            return launch_pass_hg<D, T, PASS, 4>(p, X, Y, A1, A2, G1, G2, out16, ld_t, nq16, H, scale, sms, stream);
    }
    return launch_pass_hg<D, T, PASS, 1>(p, X, Y, A1, A2, G1, G2, out16, ld_t, nq16, H, scale, sms, stream);
}

struct Scratch2 {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch2() { if (p) scratch_free(p, s); }
};

template <int D, typename T>
f3s_status launch_bwd_tc(Plan& p, const void* Q, const void* K, const void* V, const float* O_saved,
                         const float* ml_saved, const void* dO, bool dO_lp, void* dQ, void* dK, void* dV,
                         float scale, int H, cudaStream_t stream) {
    f3s_status st = build_transpose_plan(p, stream);
    if (st != F3S_OK) return st;
    Plan& tp = *p.tplan;
    int sms = 148;
    F3S_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
    const int64_t n = p.n_rows, nd = n * H * D;
    const int64_t nq16 = (n + 15) / 16 * 16 + 16;
    Scratch2 sc;
    sc.s = stream;
    const int64_t nh2 = (n * H + 1) / 2 * 2;  // keeps the arrays after (m, l) 16-byte aligned
    const bool saved = O_saved != nullptr;      // f3s_attention_backward_saved: no forward recomputation
    const size_t bytes = (saved ? 0 : sizeof(float) * (size_t)nd + sizeof(float2) * (size_t)nh2) +
                         2 * sizeof(float) * (size_t)(H * nq16) + (dO_lp ? 0 : sizeof(T) * (size_t)nd) + 256;
    F3S_CUDA_TRY(scratch_alloc(&sc.p, bytes, stream));
    char* base = static_cast<char*>(sc.p);
    const float* Op = O_saved;
    const float* ml = ml_saved;
    float2* ld_t = reinterpret_cast<float2*>(base);
    if (!saved) {
        // 1. the forward's (m, l) and unnormalised O
        float* op = reinterpret_cast<float*>(base);
        float* mlp = op + nd;
        ld_t = reinterpret_cast<float2*>(mlp + 2 * nh2);
        AttnArgs a{&p, Q, K, V, op, scale, H, D, std::is_same<T, __half>::value ? F3S_FP16 : F3S_BF16, true, stream};
        a.ml_out = mlp;
        if ((st = launch_attention_sm100(a)) != F3S_OK) return st;
        Op = op;
        ml = mlp;
    }
    // dO in the input dtype for the tensor cores: the caller's (dO_lp), else a converted copy
    T* dO16 = dO_lp ? const_cast<T*>(static_cast<const T*>(dO)) : reinterpret_cast<T*>(ld_t + H * nq16);
    const int64_t per_block = 4 * (256 / (D / 4));  // (row, head) pairs one block covers per pass
    const int pgrid = (int)std::min<int64_t>((n * H + per_block - 1) / per_block, (int64_t)sms * 8);
    if (dO_lp)
        k_bwd_prep<D, T, true><<<pgrid, 256, 0, stream>>>(Op, reinterpret_cast<const float2*>(ml), dO, n, H, nq16,
                                                          ld_t, nullptr, saved ? 1 : 0);
    else
        k_bwd_prep<D, T><<<pgrid, 256, 0, stream>>>(Op, reinterpret_cast<const float2*>(ml), dO, n, H, nq16, ld_t,
                                                    dO16, saved ? 1 : 0);
    count_launch();
    F3S_CUDA_TRY(cudaGetLastError());
    // 2. rows: dQ
    // (the _lp entry point: gradients in the input dtype too)
    if ((st = launch_pass<D, T, 0>(p, Q, dO16, K, V, dQ, nullptr, dO_lp, ld_t, nq16, H, scale, sms, stream)) != F3S_OK)
        return st;
    // 3. columns: dV (G1), dK (G2) over A^T
    if (tp.n_rows > 0 && tp.nnz == 0) {
        const size_t es = dO_lp ? sizeof(T) : sizeof(float);
        F3S_CUDA_TRY(cudaMemsetAsync(dK, 0, es * (size_t)tp.n_rows * H * D, stream));
        F3S_CUDA_TRY(cudaMemsetAsync(dV, 0, es * (size_t)tp.n_rows * H * D, stream));
        return F3S_OK;
    }
    return launch_pass<D, T, 1>(tp, K, V, Q, dO16, dV, dK, dO_lp, ld_t, nq16, H, scale, sms, stream);
}

}  // namespace

f3s_status launch_attention_backward_tc(Plan& p, const void* Q, const void* K, const void* V, const float* O,
                                        const float* ml, const void* dO, bool dO_lp, void* dQ, void* dK, void* dV,
                                        float scale, int heads, int d, f3s_dtype dtype, cudaStream_t stream) {
    if (dtype == F3S_FP16)
        return d == 64 ? launch_bwd_tc<64, __half>(p, Q, K, V, O, ml, dO, dO_lp, dQ, dK, dV, scale, heads, stream)
                       : launch_bwd_tc<128, __half>(p, Q, K, V, O, ml, dO, dO_lp, dQ, dK, dV, scale, heads, stream);
    return d == 64 ? launch_bwd_tc<64, __nv_bfloat16>(p, Q, K, V, O, ml, dO, dO_lp, dQ, dK, dV, scale, heads, stream)
                   : launch_bwd_tc<128, __nv_bfloat16>(p, Q, K, V, O, ml, dO, dO_lp, dQ, dK, dV, scale, heads, stream);
}

}  // namespace f3s
