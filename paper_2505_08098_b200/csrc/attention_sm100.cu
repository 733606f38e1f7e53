// attention_sm100.cu — the fused 3S kernel for B200 (sm_100a).
//
// Computes, per row window k (16 query rows) and head h, Alg.1 of the paper
// re-designed for Blackwell:
//
//   * work items (window or piece of a split window, head group) in LPT order from a
//     persistent queue; one CTA per SM, warps with fixed roles;
//   * warp 0 (index): pops items, bulk-copies each chunk's column ids and 16-bit row masks (the
//     BSB bitmap) into a chunk slot and TMA-loads each item's Q_w (16 x d per head, l.5);
//   * loader warps: gather the chunk's K and V rows (sptd, l.7-8) with 16-byte cp.async into
//     128B-swizzled UMMA tiles: chunk n uses K tile n % kNK and V tile n % kNV (fixed slots, freed
//     by the MMA that read them);
//   * warp 1 (MMA1) and warp 2 (MMA2): swap-AB contractions on tcgen05 with TMEM accumulators,
//       MMA1  S^T[C x 16]  = K_c[C x d] . Q_w^T        (SDDMM, l.13; M = 128, N = 16)
//       MMA2  O^T[d x 16]  = V_c^T[d x C] . P^T[C x 16] (SpMM,  l.22; M = d,   N = 16)
//     each sleeping in mbarrier try_wait on the barriers of its next instruction;
//   * two softmax warpgroups (alternate chunks): tcgen05.ld S^T (lane = compacted column, whose
//     mask is the bitmap row of l.14), chunk row max by warp shuffles (+ a 4-warp combine), online
//     softmax in fp32 with exp2 (l.16-18), P cast to the input dtype into shared memory (l.19);
//   * correction warpgroup: folds each chunk's O^T into fp32 registers with the running rescale
//     (l.21-22) and at the item's last chunk writes O = O / l (l.24; rows with l = 0 -> 0, reading
//     c4) through a shared-memory tile and one TMA store — or a split piece's (m, l, O) partial.
//
// Everything between the gathers and the O store stays on chip.  No atomics on the
// data path: results are bitwise deterministic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "internal.h"
#include "sm100.cuh"

namespace f3s {
namespace {

using namespace sm100;

// HG = heads per chunk.  HG = 1: a chunk holds up to 128 compacted columns of one head.
// HG = 4 (d = 64, every row window at most 32 columns wide, e.g. batched small graphs): a chunk
// holds the window's columns for 4 heads, head g in tile rows / S^T lanes 32g .. 32g+31, so
// softmax warp q works on head q alone (row max within the warp) and the per-chunk pipeline
// cost is paid once per 4 heads.
// EB = bytes per input element: 2 (fp16/bf16) or 1 (fp8 e4m3: d = 128, one 128-byte panel per row).
template <int D, int HG = 1, int EB = 2>
struct Cfg {
    static_assert(HG == 1 || (HG == 4 && D == 64 && EB == 2), "head groups: d = 64 only");
    static_assert(EB == 2 || (EB == 1 && HG == 1), "fp8: one head per chunk");
    static constexpr int RB = D * EB;                // bytes of one gathered row of one head
    // 128-byte panels per gathered row of one head (fp8, d = 64: a 64-byte row in the first half of
    // one panel; the MMAs read only its K-steps)
    static constexpr int P = RB >= 128 ? RB / 128 : 1;
    static constexpr int kRowPitch = 128 * P;        // bytes between tile rows of one 8-row group panel set
    // MMA2 K-step (chunk rows per instruction): 16 for kind::f16, 32 for kind::f8f6f4; ring tiles
    // are allocated in whole K-steps
    static constexpr int kRowAlign = 32 / EB;
    static constexpr int kGroupBytes = 1024 * P;     // 8 gathered rows (one swizzle atom per panel)
    static constexpr int kMaxRows = 128;             // compacted columns per chunk at most (MMA1 M = 128)
    // two softmax warpgroups take alternate CHUNKS (chunk c -> warpgroup c % 2): every chunk's
    // softmax is relative to its own row max, so chunks of one item are independent and both
    // warpgroups stay busy on long items; the correction group merges the chunk partials
    static constexpr int kSoftmaxWGs = 2;
    // S/P/O buffers in flight (TMEM and SMEM); buffer b belongs to warpgroup b % kSoftmaxWGs
    static constexpr int kSB = 4;
    static_assert(kSB % kSoftmaxWGs == 0, "S/P/O buffers are owned by one warpgroup each");
    static constexpr int kMaxRowsBytes = (kMaxRows / 8) * kGroupBytes;  // one gathered tile (K or V) of a chunk
    // chunk slots (ids, masks, header, barriers): the index warp fills them ahead of the loaders
    static constexpr int kNS = kMaxRowsBytes >= 32 * 1024 ? 18 : 16;
    // Q tile slots (items in flight per CTA); fp8 tiles are half as large and carry half the bytes
    // per chunk, so more items are kept in flight
    static constexpr int kNQ = HG == 4 ? 6 : EB == 1 ? 8 : 4;
    static constexpr int kQBytes = 16 * kRowPitch * HG;  // HG head tiles of 16 x D
    static constexpr int kPBytes = 16 * kMaxRows * EB;
    // O staging tiles (16 x HG*D fp32) for the TMA store (head groups: one per correction group)
    static constexpr int kNO = 2;
    static constexpr int kOBytes = 16 * D * 4 * HG;
    // (Row sums l_c from the tensor core -- a ones tile times P^T in MMA2 -- were measured slower,
    // MMA2 being on the critical path; round 2, profiles/r02_ab_softmax_modes.txt.)
    // TMEM: S^T, then O^T (kSB x HG buffers of 16 columns each)
    static constexpr int kTmemO = 16 * kSB * HG;
    static constexpr int kTmemUsed = 2 * 16 * kSB * HG;
    static constexpr int kTmemCols = kTmemUsed <= 128 ? 128 : kTmemUsed <= 256 ? 256 : 512;
    static_assert(kTmemUsed <= 512, "TMEM columns");
    static constexpr int kSlotBytes = 32 + 128 * 4 + 128 * 2;  // sizeof(Slot)
    static constexpr int kCorrBytes = 352;  // sizeof(CorrSlot)
    static constexpr int kNumBars = 4 * kNS + 2 * kNQ + 5 * kSB + 2 * 16;
    // everything but the gathered tiles
    static constexpr int kFixedBytes = kNQ * kQBytes + kSB * kPBytes + kNO * kOBytes + kNS * kSlotBytes +
                                       kSB * 4 * 16 * 4 + kSB * kCorrBytes + kNumBars * 8 + 16;
    // Gathered tiles: fixed-size slots of one full chunk (128 rows) each, chunk n in K tile n % kNK
    // (free again once MMA1 completed) and V tile n % kNV (free once MMA2 completed).  V tiles wait
    // for the softmax and MMA2, so they take all the shared memory that is left.
    static constexpr int kNK = kMaxRowsBytes >= 32 * 1024 ? 2 : HG == 4 ? 3 : 4;
    static constexpr int kNVmax = (227 * 1024 - kNK * kMaxRowsBytes - kFixedBytes) / kMaxRowsBytes;
    static constexpr int kNV = kNVmax > 8 ? 8 : kNVmax;
    static_assert(kNV >= 2, "two V tiles at least");
    static constexpr int oK = 0;                     // K tiles, then V tiles
    static constexpr int oV = kNK * kMaxRowsBytes;
    static constexpr int kTileBytes = (kNK + kNV) * kMaxRowsBytes;
    static constexpr int oQ = kTileBytes;
    static constexpr int oP = oQ + kNQ * kQBytes;
    static constexpr int oOst = oP + kSB * kPBytes;
    static constexpr int oSlot = oOst + kNO * kOBytes;
    static constexpr int oRed = oSlot + kNS * kSlotBytes;  // float [kSB][4][16] chunk row-max partials
    static constexpr int oCorr = oRed + kSB * 4 * 16 * 4;  // CorrSlot [kSB]
    static constexpr int oBar = oCorr + kSB * kCorrBytes;
    static constexpr int oTmem = oBar + kNumBars * 8;
    static constexpr int kSmemBytes = oTmem + 16;
    static constexpr int kCtasPerSm = 1;
    // warp roles: 0 index (work queue, chunk slots, Q tiles), 1 MMA1, 2 MMA2 (each sleeping on its
    // own barriers: try_wait wakes ~60 cycles after the arrive), kLoaderWarps cp.async gather warps,
    // two softmax warpgroups, the correction warpgroup
    // gather warps: the cp.async issue rate bounds the pipeline (measured: 5-8 warps, profiles/r02_ab_*)
    static constexpr int kLoaderWarps = RB >= 256 ? 8 : 7;
    static constexpr int kMma2Warp = 2;
    static constexpr int kLoader0 = 3, kSoftmax0 = kLoader0 + kLoaderWarps, kCorr0 = kSoftmax0 + 4 * kSoftmaxWGs;
    // correction warpgroups: head-group items are single chunks with no running state, so two
    // groups take alternate chunks; one-head items merge chunks in order in one group
    static constexpr int kCorrWGs = HG == 4 ? 2 : 1;
    // head groups (one chunk per item): a Q warp loads the per-item Q tiles, so that waiting for a free
    // Q slot never holds the index warp back (one-head plans: the index warp loads them itself)
    static constexpr int kQWarp = HG > 1 ? kCorr0 + 4 * kCorrWGs : -1;
    static constexpr int kThreads = 32 * (kCorr0 + 4 * kCorrWGs + (HG > 1 ? 1 : 0));
    static constexpr int kBatch = 8;                 // items fetched per queue round trip
    static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");
};

template <int D, int HG, int EB = 2> struct Bars {
    using C = Cfg<D, HG, EB>;
    __host__ __device__ static constexpr int idxfull(int s) { return s; }
    __host__ __device__ static constexpr int kfull(int s) { return C::kNS + s; }
    __host__ __device__ static constexpr int vfull(int s) { return 2 * C::kNS + s; }
    __host__ __device__ static constexpr int empty(int s) { return 3 * C::kNS + s; }
    __host__ __device__ static constexpr int qfull(int q) { return 4 * C::kNS + q; }
    __host__ __device__ static constexpr int qempty(int q) { return 4 * C::kNS + C::kNQ + q; }
    static constexpr int kB0 = 4 * C::kNS + 2 * C::kNQ;
    __host__ __device__ static constexpr int sfull(int b) { return kB0 + b; }
    __host__ __device__ static constexpr int pfull(int b) { return kB0 + C::kSB + b; }
    __host__ __device__ static constexpr int ofull(int b) { return kB0 + 2 * C::kSB + b; }
    __host__ __device__ static constexpr int pempty(int b) { return kB0 + 3 * C::kSB + b; }
    // S^T buffer b may be overwritten by MMA1: its owner warpgroup's 4 warps read it (and the
    // row-max partials) for the buffer's previous chunk
    __host__ __device__ static constexpr int sfree(int b) { return kB0 + 4 * C::kSB + b; }
    // gathered tile slots: K tile t free (MMA1 that read it completed), V tile t free (MMA2)
    __host__ __device__ static constexpr int ktfree(int t) { return kB0 + 5 * C::kSB + t; }
    __host__ __device__ static constexpr int vtfree(int t) { return kB0 + 5 * C::kSB + 16 + t; }
};

// One chunk of one work item: written by the index warp (header; ids/masks by cp.async.bulk);
// read by the loader, MMA and softmax warps.
struct __align__(16) Slot {
    int32_t rw;        // row window k
    int32_t head;      // head h
    int32_t rows;      // valid compacted columns in this chunk (0 for an empty RW; < 0: stop)
    int32_t reserved0;
    int32_t qslot;
    int32_t flags;     // bit0 first chunk of item, bit1 last chunk, bit2 Q-slot phase, bits 8..31 split:
                       // 0, or 1 + global piece index of a split row window (Plan::meta_sub)
    int32_t reserved1, reserved2;
    int32_t cols[128];     // gathered row ids (tail repeats the last column)
    uint16_t masks[128];   // 16-bit row masks (bitmap)
};
// softmax -> correction hand-off for one chunk (one per S/P/O buffer)
struct __align__(16) CorrSlot {
    float m[16];         // the chunk's row max m_c (log2 units, floored; Alg.1 l.16)
    float lpart[4][16];  // per-warp partial row sums of the chunk's E = 2^(S - m_c) (l.17; reading c7)
    int32_t rows, flags, rw, head;
    uint64_t t_s, t_p;   // F3S_TRACE stamps of the softmax group (written out by the correction group)
};
template <int HG> using CorrSlotT = CorrSlot;

static_assert(sizeof(CorrSlot) == Cfg<64>::kCorrBytes && sizeof(Slot) == Cfg<64>::kSlotBytes, "layout");

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

template <typename T> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) { return pack_f16x2(lo, hi); }
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) { return pack_bf16x2(lo, hi); }

template <typename T> __device__ __forceinline__ float round_to(float v);  // v rounded RNE to T, as a float
template <> __device__ __forceinline__ float round_to<__half>(float v) { return __half2float(__float2half_rn(v)); }
template <> __device__ __forceinline__ float round_to<__nv_bfloat16>(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
template <> __device__ __forceinline__ float round_to<__nv_fp8_e4m3>(float v) { return v; }

// Running row max starts at a finite floor instead of -inf so that every exponent is well
// defined without branches: 2^(floor - m) = 0 for a real m, 2^(-inf - m) = 0 for masked scores,
// and a row with no entry in a chunk keeps m_c = floor and an all-zero E (reading c5).
constexpr float kMFloor = -8.5e37f;

// kPart: head-group kernel in partial mode (unnormalised O and per-head (m, l); f3s_attention_partial)
template <int D, typename T, bool kDiag, int HG, bool kPart = false>
__global__ void __launch_bounds__(Cfg<D, HG, (int)sizeof(T)>::kThreads, Cfg<D, HG, (int)sizeof(T)>::kCtasPerSm)
k_f3s_sm100(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO, const int4* __restrict__ meta,
            const int32_t* __restrict__ kcols, const uint16_t* __restrict__ kmasks,
            int32_t* __restrict__ counter, int32_t n_items, int32_t H, int64_t ldkv,
            const uint8_t* __restrict__ Kg, const uint8_t* __restrict__ Vg, float scale_log2,
            uint64_t* __restrict__ trace, int32_t trace_chunks, int32_t expt_arg,
            float* __restrict__ scratch, float2* __restrict__ ml_out, int32_t n_rows, float* __restrict__ Og,
            int32_t heavy_items, int32_t ml_norm) {
    constexpr int EB = (int)sizeof(T);
    using C = Cfg<D, HG, EB>;
    using B = Bars<D, HG, EB>;
    constexpr int chunk_rows = C::kMaxRows;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sb = smem_u32(smem);
    if (sb & 1023) __trap();  // swizzled tiles need 1024-byte alignment
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // F3S_TRACE: stamps 8 (kernel entry) and 9 (setup done) of the CTA's first chunk record
    if (kDiag && trace != nullptr && trace_chunks > 0 && threadIdx.x == 0)
        trace[(size_t)blockIdx.x * trace_chunks * 16 + 8] = globaltimer_ns();
    auto bar = [&](int i) -> uint32_t { return sb + C::oBar + 8u * i; };
    Slot* slots = reinterpret_cast<Slot*>(smem + C::oSlot);
    CorrSlotT<HG>* corr = reinterpret_cast<CorrSlotT<HG>*>(smem + C::oCorr);
    // Sensitivity experiments exist only in the diagnostics instantiation (f3s_attention_trace
    // with trace_chunks < 0; results are wrong): bit0 no exp work in the softmax, bit1 no MMA2,
    // bit2 no MMA1, bit3 no K/V gathers, bit5 no S load / row max, bit6 no O stores, bit7 no
    // correction work.  The product kernel (kDiag = false) compiles every test away.
    const int32_t expt = kDiag ? expt_arg : 0;
    // F3S_TRACE: per CTA and chunk, globaltimer stamps of the pipeline events
    // [0 slot written, 1 gathers issued, 2 MMA1 issued, 3 S seen, 4 P written, 5 MMA2 issued, 6 O seen, 7 item stored]
    auto stamp = [&](int32_t c, int ev) {
        if (kDiag && trace != nullptr && c < trace_chunks)
            trace[((size_t)blockIdx.x * trace_chunks + c) * 16 + ev] = globaltimer_ns();
    };
    // profile mode (trace_chunks == 0): each role accumulates SM cycles spent per phase in
    // registers and writes trace[cta][64] once at the end (no stores on the hot path)
    const bool prof = kDiag && trace != nullptr && trace_chunks == 0;
    uint32_t pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t pt0 = prof ? (uint32_t)clock() : 0;
    auto lap = [&](int k) {  // charge the cycles since the previous lap to counter k
        if (prof) {
            const uint32_t t = (uint32_t)clock();
            pc[k] += t - pt0;
            pt0 = t;
        }
    };
    auto prof_flush = [&](int base) {  // base in units of roles: 8 counters each
        if (prof)
            for (int k = 0; k < 8; ++k) trace[(size_t)blockIdx.x * 64 + base * 8 / 6 + k] = (uint64_t)pc[k];
    };

    // ---- setup -------------------------------------------------------------------------------
    // Tile rows that no gather of the current chunk overwrites (past its last column) are read by
    // the MMAs with weight 0 (masked / P = 0): they must be finite, so every tile starts zeroed and
    // only ever holds gathered input rows.
    for (int i = threadIdx.x; i < C::kTileBytes / 16; i += blockDim.x)
        reinterpret_cast<int4*>(smem + C::oK)[i] = make_int4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kNS; ++s) {
            mbar_init(bar(B::idxfull(s)), 1);
            mbar_init(bar(B::kfull(s)), 32 * C::kLoaderWarps);  // one cp.async completion per loader lane
            mbar_init(bar(B::vfull(s)), 32 * C::kLoaderWarps);
            mbar_init(bar(B::empty(s)), 1);   // slot retired: MMA2 done
        }
        for (int t = 0; t < C::kNK; ++t) mbar_init(bar(B::ktfree(t)), 1);
        for (int t = 0; t < C::kNV; ++t) mbar_init(bar(B::vtfree(t)), 1);
        for (int q = 0; q < C::kNQ; ++q) {
            mbar_init(bar(B::qfull(q)), 1);
            mbar_init(bar(B::qempty(q)), 1);
        }
        for (int b = 0; b < C::kSB; ++b) {
            mbar_init(bar(B::sfull(b)), 1);
            mbar_init(bar(B::pfull(b)), 128);
            mbar_init(bar(B::ofull(b)), 1);
            mbar_init(bar(B::pempty(b)), 128);
            mbar_init(bar(B::sfree(b)), 4);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmO);
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
    if (kDiag && trace != nullptr && trace_chunks > 0 && threadIdx.x == 0)
        trace[(size_t)blockIdx.x * trace_chunks * 16 + 9] = globaltimer_ns();

    if (warp == 0) {
        // ===== index warp: work queue (LPT order) -> chunk slots and Q tiles ==============
        // kBatch lanes each take one item per queue round trip; per chunk one lane issues two
        // bulk copies (column ids, masks) straight into the slot, and at an item's first chunk the
        // TMA load of Q_w (16 x d per head, Alg.1 l.5) into the item's Q slot.
        int32_t seq = 0, qseq = 0, last = 0;
        bool done = false;
        // claim batch: kBatch items per queue round trip, fewer when the problem has under
        // 4 kBatch items per CTA (a small graph would otherwise run on n_items / kBatch CTAs)
        const int batch = max(1, min(C::kBatch, n_items / (4 * (int)gridDim.x)));
        while (!done) {
            // items of the LPT list's heavy prefix are claimed one per round trip, the rest
            // `batch` at a time (the claim is per lane: consecutive indices, one CTA)
            const int nclaim = last < heavy_items ? 1 : batch;
            int32_t it = 0x7FFFFFFF;
            int4 mt = make_int4(0, 0, 0, 0);
            if (lane < nclaim) {
                it = atomicAdd(counter, 1);
                if (it < n_items) mt = __ldg(meta + it / (H / HG));
            }
            __syncwarp();
            last = __shfl_sync(0xffffffffu, it, nclaim - 1);
            if (lane == 0) lap(1);
            for (int b = 0; b < nclaim; ++b) {
                const int32_t itb = __shfl_sync(0xffffffffu, it, b);
                const int32_t k = __shfl_sync(0xffffffffu, mt.x, b);
                const int32_t cb8 = __shfl_sync(0xffffffffu, mt.y, b);
                const int32_t w = __shfl_sync(0xffffffffu, mt.z, b);
                const int32_t sp = __shfl_sync(0xffffffffu, mt.w, b);
                if (itb >= n_items) { done = true; continue; }
                const int32_t h = (itb - (itb / (H / HG)) * (H / HG)) * HG;  // (first) head
                const int nch = w > 0 ? (w + chunk_rows - 1) / chunk_rows : 1;
                const int qs = qseq % C::kNQ;
                const int qph = (qseq / C::kNQ) & 1;
                if (HG == 1 && lane == 0) {  // Alg.1 l.5: Q_i of the item (the slot's previous item has left MMA1)
                    mbar_wait(bar(B::qempty(qs)), qph ^ 1);
                    mbar_arrive_expect_tx(bar(B::qfull(qs)), C::kQBytes);
#pragma unroll
                    for (int g = 0; g < HG; ++g)
#pragma unroll
                        for (int pp = 0; pp < C::P; ++pp)
                            tma_load_2d(sb + C::oQ + qs * C::kQBytes + g * 16 * C::kRowPitch + pp * 2048, &tmQ,
                                        bar(B::qfull(qs)), (h + g) * D + (128 / EB) * pp, 16 * k);
                }
                for (int j = 0; j < nch; ++j) {
                    const int rows = w > 0 ? min(chunk_rows, w - chunk_rows * j) : 0;
                    const int s = seq % C::kNS;
                    if (lane == 0) {
                        mbar_wait(bar(B::empty(s)), ((seq / C::kNS) & 1) ^ 1);
                        lap(0);
                        Slot& sl = slots[s];
                        sl.rw = k;
                        sl.head = h;
                        sl.rows = rows;
                        sl.qslot = qs;
                        sl.flags = (j == 0 ? 1 : 0) | (j == nch - 1 ? 2 : 0) | (qph << 2) | (sp << 8);
                        const uint32_t fb = bar(B::idxfull(s));
                        if (rows > 0) {
                            const uint32_t r8 = (uint32_t)((rows + 7) & ~7);
                            mbar_arrive_expect_tx(fb, r8 * 6u);
                            bulk_g2s(smem_u32(sl.cols), kcols + cb8 + chunk_rows * j, r8 * 4u, fb);
                            bulk_g2s(smem_u32(sl.masks), kmasks + cb8 + chunk_rows * j, r8 * 2u, fb);
                        } else {
                            mbar_arrive(fb);
                        }
                        stamp(seq, 0);
                        lap(2);
                    }
                    ++seq;
                }
                ++qseq;
            }
        }
        if (lane == 0) {
            // one stop marker per softmax warpgroup (each walks only its own chunk parity); the
            // producer, loaders and MMA warps stop at the first.  rows = -1 - w.
            for (int w = 0; w < C::kSoftmaxWGs; ++w, ++seq) {
                const int s = seq % C::kNS;
                mbar_wait(bar(B::empty(s)), ((seq / C::kNS) & 1) ^ 1);
                slots[s].rows = -1 - w;
                mbar_arrive(bar(B::idxfull(s)));
            }
            prof_flush(0);
        }
        __syncwarp();
    } else if (HG > 1 && warp == C::kQWarp) {
        // ===== Q warp (head groups): Alg.1 l.5, the item's Q tiles by TMA once its Q slot's previous
        // item has left MMA1; walks the chunk slots in order and loads at each item's first chunk
        if (lane == 0) {
            for (int32_t seq = 0;; ++seq) {
                const int s = seq % C::kNS;
                mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);
                const Slot& sl = slots[s];
                const int rows = sl.rows, flags = sl.flags;
                if (rows < 0) break;
                if (!(flags & 1)) continue;
                const int qs = sl.qslot, qph = (flags >> 2) & 1, k = sl.rw, h = sl.head;
                mbar_wait(bar(B::qempty(qs)), qph ^ 1);
                mbar_arrive_expect_tx(bar(B::qfull(qs)), C::kQBytes);
#pragma unroll
                for (int g = 0; g < HG; ++g)
#pragma unroll
                    for (int pp = 0; pp < C::P; ++pp)
                        tma_load_2d(sb + C::oQ + qs * C::kQBytes + g * 16 * C::kRowPitch + pp * 2048, &tmQ,
                                    bar(B::qfull(qs)), (h + g) * D + (128 / EB) * pp, 16 * k);
            }
        }
        __syncwarp();
    } else if (warp >= C::kLoader0 && warp < C::kLoader0 + C::kLoaderWarps) {
        // ===== loader warps: gather the K and V rows of each chunk (Alg.1 l.8) ===================
        // Lane l of a warp copies 16-byte piece (l % pieces) of one gathered row straight into the
        // 128B-swizzled UMMA layout; the rows of a chunk are dealt round-robin to the warps.
        // Each lane arrives on the chunk's K/V barriers when its own copies have landed.
        constexpr int kPieces = C::RB / 16;
        constexpr int kRowsPerOp = 32 / kPieces;
        const int lw = warp - C::kLoader0;
        const int piece = lane % kPieces, rsub = lane / kPieces;
        const int pnl = piece >> 3, cc = piece & 7;
        const int64_t ldb = ldkv;  // bytes between consecutive K (and V) rows
        int32_t seq = 0;
        for (;;) {
            const int s = seq % C::kNS;
            mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);  // the chunk's ids have landed
            if (lw == 0 && lane == 0) stamp(seq, 10);
            const Slot& sl = slots[s];
            const int rows = sl.rows;
            const uint32_t kfb = bar(B::kfull(s)), vfb = bar(B::vfull(s));
            if (rows < 0) {
                mbar_arrive(kfb);
                mbar_arrive(vfb);
                break;
            }
            const int h = sl.head;
            const int tk = seq % C::kNK, tv = seq % C::kNV;
            const uint32_t kt = sb + C::oK + tk * C::kMaxRowsBytes + pnl * 1024;
            const uint32_t vt = sb + C::oV + tv * C::kMaxRowsBytes + pnl * 1024;
            const uint8_t* kbase = Kg + (int64_t)h * C::RB + piece * 16;
            const uint8_t* vbase = Vg + (int64_t)h * C::RB + piece * 16;
            // HG = 1: tile row r = compacted column r.  HG = 4: tile row 32g + r = column r of head h + g.
            const int ops = (expt & 8) ? 0 : (HG == 1 ? (rows + kRowsPerOp - 1) / kRowsPerOp : C::kMaxRows / kRowsPerOp);
            mbar_wait(bar(B::ktfree(tk)), ((seq / C::kNK) & 1) ^ 1);
            mbar_wait(bar(B::vtfree(tv)), ((seq / C::kNV) & 1) ^ 1);
            // all of this lane's row ids first (independent shared loads), then the copies
            constexpr int kIters = (C::kMaxRows / kRowsPerOp + C::kLoaderWarps - 1) / C::kLoaderWarps;
            int64_t src[kIters];
            uint32_t dst[kIters];
            bool ok[kIters];
#pragma unroll
            for (int i = 0; i < kIters; ++i) {
                const int t = lw + i * C::kLoaderWarps;
                const int tr = t * kRowsPerOp + rsub;  // tile row
                const int r = HG == 1 ? tr : (tr & 31);
                ok[i] = t < ops && r < rows;
                const int64_t j = ok[i] ? sl.cols[r] : 0;
                src[i] = j * ldb + (HG == 1 ? 0 : (int64_t)(tr >> 5) * C::RB);
                dst[i] = (uint32_t)(tr >> 3) * C::kGroupBytes + (uint32_t)(tr & 7) * 128 + (uint32_t)((cc ^ (tr & 7)) << 4);
            }
#pragma unroll
            for (int i = 0; i < kIters; ++i)
                if (ok[i]) cp_async_16(kt + dst[i], kbase + src[i]);
            cp_async_mbar_arrive(kfb);
#pragma unroll
            for (int i = 0; i < kIters; ++i)
                if (ok[i]) cp_async_16(vt + dst[i], vbase + src[i]);
            cp_async_mbar_arrive(vfb);
            if (lw == 0 && lane == 0) stamp(seq, 1);
            ++seq;
        }
    } else if (warp == 1 || warp == C::kMma2Warp) {
        // ===== MMA issuers: warp 1 issues MMA1 (SDDMM), warp kMma2Warp MMA2 (SpMM) ====================
        // Each walks the chunks in order and sleeps in try_wait on the barriers of its next
        // instruction.  Whole warps run the loops on warp-uniform values; one elected lane issues
        // (sm100.cuh: mma_f16_ss_warp).  The cp.async-written K/V tiles need no proxy fence here
        // (the mbarrier completion of cp.async orders them, as in CUTLASS's SM100 cp.async
        // mainloop); P is fenced by its writers before pfull.
        constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
        if (warp == 1) {
            constexpr uint32_t idesc1 = idesc_f16(fmt, 0, 0, 128, 16);  // S^T = K_c . Q_w^T
            const uint64_t dK = smem_desc_sw128(0, 16, C::kGroupBytes);
            const uint64_t dQ = smem_desc_sw128(0, 16, 1024);
            for (int32_t n1 = 0;; ++n1) {
                const int s = n1 % C::kNS, b = n1 % C::kSB;
                mbar_wait(bar(B::kfull(s)), (n1 / C::kNS) & 1);  // K_c landed
                if (lane == 0) stamp(n1, 11);
                const Slot& sl = slots[s];
                const int rows = sl.rows, flags = sl.flags, qslot = sl.qslot;
                if (rows < 0) break;
                mbar_wait(bar(B::sfree(b)), ((n1 / C::kSB) & 1) ^ 1);  // owner read chunk n1 - kSB
                if (flags & 1) mbar_wait(bar(B::qfull(qslot)), (flags >> 2) & 1);
                tc_fence_after();
                const uint64_t a0 = dK + ((sb + C::oK + (n1 % C::kNK) * C::kMaxRowsBytes) >> 4);
                const uint64_t b0 = dQ + ((sb + C::oQ + qslot * C::kQBytes) >> 4);
                if (rows > 0 && !(expt & 4)) {
                    if constexpr (HG > 1) {
                        // head groups (d = 64): the HG Q tiles are one [16 HG x 64] K-major tile, so one
                        // N = 16 HG MMA per K-step gives S^T of every tile row against every head's
                        // rows; lanes 32g .. 32g+31 (head g's tile rows) are read back from columns
                        // 16g .. 16g+15 only -- the products with the other heads' Q are never read
                        constexpr uint32_t idesc1g = idesc_f16(fmt, 0, 0, 128, 16 * HG);
#pragma unroll
                        for (int kk = 0; kk < C::RB / 32; ++kk)
                            mma_f16_ss_warp(tmem + b * HG * 16, a0 + ((kk * 32) >> 4), b0 + ((kk * 32) >> 4), idesc1g,
                                            kk > 0 ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < C::RB / 32; ++kk) {  // K-steps of 32 bytes
                            const uint64_t ad = a0 + (((kk >> 2) * 1024 + (kk & 3) * 32) >> 4);
                            const uint64_t bd = b0 + (((kk >> 2) * 2048 + (kk & 3) * 32) >> 4);
                            if (EB == 1) mma_f8_ss_warp(tmem + b * 16, ad, bd, idesc1, kk > 0 ? 1u : 0u);
                            else mma_f16_ss_warp(tmem + b * 16, ad, bd, idesc1, kk > 0 ? 1u : 0u);
                        }
                    }
                }
                mma_commit_warp(bar(B::sfull(b)));
                mma_commit_warp(bar(B::ktfree(n1 % C::kNK)));
                if (flags & 2) mma_commit_warp(bar(B::qempty(qslot)));
                if (lane == 0) stamp(n1, 2);
            }
        } else {
            // O^T = V_c^T . P^T: A (V_c) MN-major; B (P^T) MN-major with a 32-byte swizzle for
            // 16-bit P, K-major [16 x 128 bytes] with the 128-byte swizzle for fp8 P (8-bit
            // MN-major B would need 16-byte rows)
            constexpr uint32_t idesc2 = idesc_f16(fmt, 1, EB == 2 ? 1 : 0, D, 16);
            const uint64_t dV = smem_desc_sw128(0, 1024, C::kGroupBytes);
            const uint64_t dP = EB == 2 ? smem_desc_sw32(0, 4096, 256) : smem_desc_sw128(0, 16, 1024);
            for (int32_t n2 = 0;; ++n2) {
                const int s = n2 % C::kNS, b = n2 % C::kSB;
                mbar_wait(bar(B::kfull(s)), (n2 / C::kNS) & 1);  // slot of chunk n2 filled
                const int rows = slots[s].rows;
                if (rows < 0) break;
                mbar_wait(bar(B::pfull(b)), (n2 / C::kSB) & 1);  // P_c written
                if (lane == 0) stamp(n2, 13);
                mbar_wait(bar(B::vfull(s)), (n2 / C::kNS) & 1);  // V_c landed
                if (lane == 0) stamp(n2, 14);
                tc_fence_after();
                if (rows > 0 && !(expt & 2)) {
                    const uint64_t a0 = dV + ((sb + C::oV + (n2 % C::kNV) * C::kMaxRowsBytes) >> 4);
                    const uint64_t b0 = dP + ((sb + C::oP + b * C::kPBytes) >> 4);
                    const int nsteps = (rows + C::kRowAlign - 1) / C::kRowAlign;
                    if (EB == 1) {
                        for (int st = 0; st < nsteps; ++st)  // 32 chunk rows = 4 row groups, 32 bytes of a P row
                            mma_f8_ss_warp(tmem + C::kTmemO + b * 16, a0 + ((st * 4 * C::kGroupBytes) >> 4),
                                           b0 + ((st * 32) >> 4), idesc2, st > 0 ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int g = 0; g < HG; ++g)  // head g: tile rows / P^T columns 32g .. (HG > 1)
                            for (int st = 0; st < nsteps; ++st)
                                mma_f16_ss_warp(tmem + C::kTmemO + (b * HG + g) * 16,
                                                a0 + ((g * 4 * C::kGroupBytes + st * 2 * C::kGroupBytes) >> 4),
                                                b0 + ((g * 1024 + st * 512) >> 4), idesc2, st > 0 ? 1u : 0u);
                    }
                }
                mma_commit_warp(bar(B::ofull(b)));
                mma_commit_warp(bar(B::vtfree(n2 % C::kNV)));
                mma_commit_warp(bar(B::empty(s)));
                if (lane == 0) stamp(n2, 5);
                __syncwarp();
            }
        }
        __syncwarp();
    } else if (warp < C::kCorr0) {
        // ===== softmax warpgroups ====================================================
        // Warpgroup wg takes chunks c = wg, wg + 2, ... (every chunk of every item).  Per chunk
        // (Alg.1 l.14-19): masked scores, the chunk's row max m_c (l.16), E = 2^(S - m_c) (l.17),
        // E cast to the input dtype for MMA2 (l.19), and the per-warp partial row sums of the
        // unrounded E (l.18).  Relative to m_c rather than the running max, every chunk is
        // independent of the item's earlier chunks; the correction group applies the rescaling
        // of l.18/l.21 when it merges the chunk into the running (m, l, O).
        const int q = warp & 3;          // TMEM lane quadrant this warp may access
        const int p = 32 * q + lane;     // compacted column of the chunk (S^T lane)
        const int wg = (warp - C::kSoftmax0) >> 2;
        const uint32_t tl = (uint32_t)(32 * q) << 16;
        float* red = reinterpret_cast<float*>(smem + C::oRed);
        for (int32_t seq = wg;; seq += C::kSoftmaxWGs) {
            const int s = seq % C::kNS;
            const int b = seq % C::kSB;
            const uint32_t bph = (seq / C::kSB) & 1;
            // the slot header and masks (idxfull: the index warp's writes and bulk copies);
            // the slot cannot be retired before MMA2 has this chunk's P
            mbar_wait(bar(B::idxfull(s)), (seq / C::kNS) & 1);
            if (p == 0) lap(0);
            const Slot& sl = slots[s];
            const int rows = sl.rows;
            if (rows < 0) {  // forward the stop to the correction group(s) that walk this chunk's parity
                if (rows == -1 || (C::kCorrWGs == 2 && rows == -2)) {
                    mbar_wait(bar(B::pempty(b)), bph ^ 1);
                    if (p == 0) corr[b].rows = -1;
                    mbar_arrive(bar(B::pfull(b)));
                }
                if (p == 0) prof_flush(18);
                break;
            }
            const int flags = sl.flags;
            // S^T lane p <-> compacted column p (HG = 1), or column `lane` of head q (HG = 4)
            const int col = HG == 1 ? p : lane;
            const uint32_t mask = col < rows ? (uint32_t)sl.masks[col] : 0u;
            const int rw = sl.rw, hd = sl.head;
            mbar_wait(bar(B::sfull(b)), bph);
            tc_fence_after();
            uint64_t t_s = 0;
            if (kDiag && p == 0) { t_s = globaltimer_ns(); lap(1); }
            float x[16];
            if (expt & 32) {
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = 0.f;
            } else {
                tmem_ld_32x32b_x16(tmem + tl + (b * HG + (HG > 1 ? q : 0)) * 16, x);
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = ((mask >> i) & 1u) ? x[i] * scale_log2 : -INFINITY;  // Alg.1 l.14
            }
            // chunk row max (Alg.1 l.16)
            float cm[16];
            float mrow = kMFloor;  // HG = 1, lanes 0..15: the chunk max of row `lane` (reading c5 floor)
            float rm_hg = kMFloor;  // HG = 4, lane 2i: row i's max of the warp's head
            if constexpr (HG == 1) {
                // the warp's 32 columns: one redux.sync.max per row (uniform datapath), then the
                // 4-warp combine through shared memory; lane i < 16 finishes row i and broadcasts
                float mine = -INFINITY;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float wm = (expt & 32) ? 0.f : redux_max_f32(x[i]);
                    mine = (lane & 15) == i ? wm : mine;
                }
                if (lane < 16) red[(b * 16 + lane) * 4 + q] = mine;
                if (p == 0) lap(2);
                named_bar_sync(1 + wg, 128);
                if (lane < 16) {
                    const float4 r = reinterpret_cast<const float4*>(red)[b * 16 + lane];
                    mrow = fmaxf(fmaxf(fmaxf(r.x, r.y), fmaxf(r.z, r.w)), kMFloor);
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) cm[i] = __shfl_sync(0xffffffffu, mrow, i);
            } else {  // the warp holds all columns of its head: lane 2i has row i's max
                rm_hg = (expt & 32) ? 0.f : rowreduce16(x, lane, OpMax());
#pragma unroll
                for (int i = 0; i < 16; ++i) cm[i] = __shfl_sync(0xffffffffu, rm_hg, 2 * i);
            }
            // S^T_b and red[b] are read: MMA1 may refill buffer b (its next chunk is this
            // warpgroup's own, so red[b] is rewritten only after this chunk's combine)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(B::sfree(b)));
            if (p == 0) lap(3);
            // fp8 P: E scaled by 2^8 (exponent offset) so that [0, 1] lands in e4m3's normal range
            // [2^-6, 448] down to 2^-14; l sums the same scaled values, so O / l is unchanged
            auto pexp = [](float v) { return EB == 1 ? ex2(v + 8.f) : ex2(v); };
            float pv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                cm[i] = fmaxf(kMFloor, cm[i]);                    // m_c (reading c5)
                pv[i] = (expt & 1) ? x[i] : pexp(x[i] - cm[i]);   // E = e^{S - m_c} (l.17); 0 where masked
            }
            // this warp's part of the row sums (l.18) of the P that MMA2 multiplies: the rounded
            // 16-bit P (reading c7), or fp8's unrounded E (reading c24)
            float pr[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pr[i] = EB == 1 ? pv[i] : round_to<T>(pv[i]);
            const float rl = rowreduce16(pr, lane, OpAdd());
            if (p == 0) lap(6);
            // P_b / corr_b are free once the correction group consumed chunk seq - kSB
            mbar_wait(bar(B::pempty(b)), bph ^ 1);
            if (p == 0) { lap(4); stamp(seq, 15); }
            if constexpr (EB == 1) {
                // E cast to e4m3 (satfinite, round to nearest even) into the K-major 128B-swizzled
                // [16 x 128] B tile: byte p of row i, 16-byte chunk (p >> 4) ^ (i & 7)
                uint8_t* pt = smem + C::oP + b * C::kPBytes + (p & 15);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    pt[(i >> 3) * 1024 + (i & 7) * 128 + ((((p >> 4) ^ (i & 7)) & 7) << 4)] =
                        (uint8_t)__nv_cvt_float_to_fp8(pv[i], __NV_SATFINITE, __NV_E4M3);
            } else {
                // E cast to the input dtype (l.19): P^T is the MN-major B operand of MMA2 with a
                // 32-byte swizzle: compacted column p owns one 32-byte row (its 16 query rows), 8
                // rows per 256-byte atom, the two 16-byte halves swapped when bit 2 of p is set
                uint4* prow = reinterpret_cast<uint4*>(smem + C::oP + b * C::kPBytes + (p >> 3) * 256 + (p & 7) * 32);
                const int sw = (p >> 2) & 1;
                const uint4 lo = make_uint4(pack2<T>(pv[0], pv[1]), pack2<T>(pv[2], pv[3]), pack2<T>(pv[4], pv[5]),
                                            pack2<T>(pv[6], pv[7]));
                const uint4 hi = make_uint4(pack2<T>(pv[8], pv[9]), pack2<T>(pv[10], pv[11]), pack2<T>(pv[12], pv[13]),
                                            pack2<T>(pv[14], pv[15]));
                prow[sw] = lo;
                prow[sw ^ 1] = hi;
            }
            if (!(lane & 1)) corr[b].lpart[q][(lane >> 1) & 15] = rl;
            if (HG == 1 && q == 0 && lane < 16) corr[b].m[lane] = mrow;
            if constexpr (HG > 1 && kPart) {  // partial / training outputs: head q's (m, l) of each row
                const int r = lane >> 1;
                if (!(lane & 1) && 16 * rw + r < n_rows)
                    ml_out[(int64_t)(16 * rw + r) * H + hd + q] =
                        rows > 0 ? make_float2(fmaxf(kMFloor, rm_hg), rl) : make_float2(kMFloor, 0.f);
            }
            if (p == 0) {
                reinterpret_cast<int4*>(&corr[b].rows)[0] = make_int4(rows, flags, rw, hd);
                if (kDiag) {
                    corr[b].t_s = t_s;
                    corr[b].t_p = globaltimer_ns();
                }
            }
            if (p == 0) lap(7);
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(bar(B::pfull(b)));
            if (p == 0) lap(5);
        }
    } else {
        // ===== correction / epilogue warpgroup =======================================
        // Chunks in order: merge chunk c's (m_c, l_c, O_c = E_c V_c) into the item's running
        // (m, l, O) with the rescaling of Alg.1 l.18/l.21:
        //   M = max(m, m_c),  l = 2^(m - M) l + 2^(m_c - M) l_c,  O = 2^(m - M) O + 2^(m_c - M) O_c
        // and at the item's last chunk write O = O / l (l.24; rows with l = 0 -> 0, reading c4)
        // through a shared-memory tile and one TMA store, or a split piece's (m, l, O) partial.
        // O^T lives in fp32 registers: thread (warp q, lane) holds one feature for the 16 rows.
        const int q = warp & 3;
        const uint32_t tl = (uint32_t)(32 * q) << 16;
        const int ri = lane & 15;        // the row whose statistics this lane keeps (lanes 16..31 mirror)
        (void)Og;
        float oacc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) oacc[i] = 0.f;
        float m_run = kMFloor, l_run = 0.f;
        int32_t item = 0;
        const int cw = (warp - C::kCorr0) >> 2;  // correction group (head groups: alternate chunks)
        for (int32_t seq = cw;; seq += C::kCorrWGs) {
            const int b = seq % C::kSB;
            const uint32_t bph = (seq / C::kSB) & 1;
            mbar_wait(bar(B::pfull(b)), bph);
            const bool lead = lane == 0 && q == 0;
            if (lead) lap(0);
            const int4 info = reinterpret_cast<const int4*>(&corr[b].rows)[0];
            const int rows = info.x, flags = info.y, rw = info.z, hd = info.w;
            const int split = flags >> 8;
            if (rows < 0) {
                if (lead) prof_flush(24);
                break;
            }
            // the chunk's O_c^T arrives in TMEM
            mbar_wait(bar(B::ofull(b)), bph);
            tc_fence_after();
            if (lead) {
                if (kDiag && trace != nullptr && seq < trace_chunks) {
                    trace[((size_t)blockIdx.x * trace_chunks + seq) * 16 + 3] = corr[b].t_s;
                    trace[((size_t)blockIdx.x * trace_chunks + seq) * 16 + 4] = corr[b].t_p;
                }
                stamp(seq, 6);
                lap(1);
            }
            if constexpr (HG > 1) {
                // head groups: one chunk per item (every window <= 32 columns), so O_g = O^T_g / l_g
                // for each head g of the group (warp g's row sums are head g's), staged as one
                // [16 x HG*D] tile per correction group and stored by one TMA
                float* ost = reinterpret_cast<float*>(smem + C::oOst + cw * C::kOBytes);
                const bool wlead = lane == 0 && q == 0;
                if (wlead) bulk_wait_group_read<0>();  // this group's previous store has read the tile
                named_bar_sync(1 + C::kSoftmaxWGs + cw, 128);
                const bool has = lane < 16;           // O^T lane -> feature 16q + lane (M = 64 layout)
                const int f = 16 * q + lane;
#pragma unroll 1
                for (int g = 0; g < HG; ++g) {
                    float ov[16];
                    tmem_ld_32x32b_x16(tmem + tl + C::kTmemO + (b * HG + g) * 16, ov);
                    const float4* l4 = reinterpret_cast<const float4*>(corr[b].lpart[g]);  // head g's row sums
                    if (has && (!kPart || ml_norm)) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float4 lv = l4[u];
                            const float lt[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                const int i = 4 * u + v;  // empty row (l = 0) -> 0 (reading c4)
                                ost[i * (HG * D) + g * D + f] = (rows > 0 && lt[v] > 0.f) ? ov[i] * rcp_approx(lt[v]) : 0.f;
                            }
                        }
                    } else if (has) {  // partial mode: unnormalised O (unless ml_norm); the softmax warps wrote each head's (m, l)
#pragma unroll
                        for (int i = 0; i < 16; ++i) ost[i * (HG * D) + g * D + f] = rows > 0 ? ov[i] : 0.f;
                    }
                }
                tc_fence_before();
                mbar_arrive(bar(B::pempty(b)));
                fence_proxy_async_smem();
                named_bar_sync(1 + C::kSoftmaxWGs + cw, 128);
                if (wlead) {
                    if (!(expt & 64)) tma_store_2d(&tmO, smem_u32(ost), hd * D, 16 * rw);
                    bulk_commit_group();
                    stamp(seq, 7);
                }
                ++item;
                continue;
            }
            // merge factors of row ri: O = fa * O + fb * O_c
            const float mc = corr[b].m[ri];
            const float lc = (corr[b].lpart[0][ri] + corr[b].lpart[1][ri]) + (corr[b].lpart[2][ri] + corr[b].lpart[3][ri]);
            float fa, fb;
            if (flags & 1) {  // the item's first chunk: (m, l) = (m_c, l_c)
                m_run = mc;
                l_run = lc;
                fa = 0.f;
                fb = 1.f;
            } else {
                const float M = fmaxf(m_run, mc);
                fa = ex2(m_run - M);
                fb = ex2(mc - M);
                l_run = fmaf(l_run, fa, lc * fb);
                m_run = M;
            }
            if (expt & 128) {  // diagnostics: the correction group only keeps the barrier protocol
                tc_fence_before();
                mbar_arrive(bar(B::pempty(b)));
                if (flags & 2) ++item;
                continue;
            }
            if (rows > 0) {
                float ov[16];
                tmem_ld_32x32b_x16(tmem + tl + C::kTmemO + b * 16, ov);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    oacc[i] = fmaf(oacc[i], __shfl_sync(0xffffffffu, fa, i), ov[i] * __shfl_sync(0xffffffffu, fb, i));
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) oacc[i] *= __shfl_sync(0xffffffffu, fa, i);
            }
            tc_fence_before();
            mbar_arrive(bar(B::pempty(b)));
            if (lead) lap(2);
            if (flags & 2) {
                // O_i = diag(l)^-1 O_i (l.24); empty row (l = 0) -> 0 (reading c4).  Partial mode
                // (ml_out != nullptr, f3s_attention_partial): O stays unnormalised and the row's
                // (m, l) go to ml_out, for f3s_attention_merge to combine column blocks; with
                // ml_norm (f3s_attention_fwd) O is normalised as in f3s_attention and (m, l) kept
                const float linv = (ml_out && !ml_norm) ? 1.f : l_run > 0.f ? rcp_approx(l_run) : 0.f;
                float li[16];  // 1 / l of the 16 rows, broadcast to every lane (outside the lane-divergent stores)
#pragma unroll
                for (int i = 0; i < 16; ++i) li[i] = __shfl_sync(0xffffffffu, linv, i);
                const bool has = D == 128 || lane < 16;
                const int f = D == 128 ? 32 * q + lane : 16 * q + lane;  // O^T lane -> feature (M = 64 layout)
                if (split) {
                    // piece of a split row window: leave (m, l, unnormalised O) in the scratch
                    // record of its global piece; k_split_merge combines the pieces after the
                    // kernel, in piece order (deterministic)
                    const int64_t rec_floats = 32 + 16 * D;
                    float* rec = scratch + ((int64_t)(split - 1) * H + hd) * rec_floats;
                    if (q == 0 && lane < 16) {
                        rec[lane] = m_run;
                        rec[16 + lane] = l_run;
                    }
                    if (has) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) rec[32 + i * D + f] = oacc[i];
                    }
                } else {
                    if (ml_out && q == 0 && lane < 16 && 16 * rw + lane < n_rows)
                        ml_out[(int64_t)(16 * rw + lane) * H + hd] = make_float2(m_run, l_run);
                    // O tile [16 x D] fp32 staged in shared memory and written by one TMA store
                    // (rows past n_rows of a ragged last window are clipped by the tensor map, c14)
                    const int ob = item % C::kNO;
                    float* ost = reinterpret_cast<float*>(smem + C::oOst + ob * C::kOBytes);
                    if (threadIdx.x == 32 * C::kCorr0) bulk_wait_group_read<C::kNO - 1>();  // staging tile ob free
                    named_bar_sync(1 + C::kSoftmaxWGs, 128);
                    if (has) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) ost[i * D + f] = oacc[i] * li[i];
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1 + C::kSoftmaxWGs, 128);
                    if (threadIdx.x == 32 * C::kCorr0) {
                        if (!(expt & 64)) tma_store_2d(&tmO, sb + C::oOst + ob * C::kOBytes, hd * D, 16 * rw);
                        bulk_commit_group();
                    }
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) oacc[i] = 0.f;
                if (lead) { stamp(seq, 7); lap(3); }
                ++item;
            }
        }
        if (lane == 0 && (HG > 1 ? q == 0 : threadIdx.x == 32 * C::kCorr0)) bulk_wait_group<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

// Merge of a split row window: pieces p = 0..np-1 of window k left
// (m_p, l_p, O_p) for each of its 16 rows (m in log2 units, O unnormalised); in piece order,
//   M = max_p m_p,  l = sum_p 2^(m_p - M) l_p,  O = sum_p 2^(m_p - M) O_p / l   (0 if l = 0)
// which is the online-softmax rescaling of Alg.1 l.18/l.21 applied once per piece.
template <int D>
__global__ void __launch_bounds__(256) k_split_merge(const int4* __restrict__ ginfo, const float* __restrict__ scratch,
                                                     float* __restrict__ O, int32_t H, int32_t n_rows,
                                                     float2* __restrict__ ml_out, int32_t ml_norm) {
    const int g = blockIdx.x / H, h = blockIdx.x - (blockIdx.x / H) * H;
    const int4 gi = ginfo[g];
    const int64_t rec_floats = 32 + 16 * D, stride = (int64_t)H * rec_floats;
    const float* r0 = scratch + ((int64_t)gi.x * H + h) * rec_floats;
    for (int e = threadIdx.x; e < 16 * D; e += blockDim.x) {
        const int i = e / D, f = e - (e / D) * D;
        float M = -INFINITY;
        for (int j = 0; j < gi.y; ++j) M = fmaxf(M, r0[j * stride + i]);
        float l = 0.f, acc = 0.f;
        for (int j = 0; j < gi.y; ++j) {
            const float* rj = r0 + j * stride;
            const float w = exp2f(rj[i] - M);
            l = fmaf(w, rj[16 + i], l);
            acc = fmaf(w, rj[32 + i * D + f], acc);
        }
        const int64_t row = 16 * (int64_t)gi.z + i;
        if (row >= n_rows) continue;
        if (ml_out) {  // partial mode: the window's unnormalised O (normalised: ml_norm) and its (m, l)
            O[(row * H + h) * D + f] = ml_norm ? (l > 0.f ? acc / l : 0.f) : acc;
            if (f == 0) ml_out[row * H + h] = make_float2(M, l);
        } else {
            O[(row * H + h) * D + f] = l > 0.f ? acc / l : 0.f;  // empty row -> 0 (reading c4)
        }
    }
}

}  // namespace

// Merge of column-block partials (K/V blocks that arrive one by one are processed
// as they land, each leaving the unnormalised (m, l, O) of every row): in part order
//   M = max_g m_g,  l = sum_g 2^(m_g - M) l_g,  O = sum_g 2^(m_g - M) O_g / l   (0 if l = 0),
// the rescaling of Alg.1 l.18/l.21 applied once per block.  One warp per (row, head); fixed order,
// so the result is deterministic.
__global__ void __launch_bounds__(256) k_parts_merge(int32_t parts, const float* __restrict__ Op,
                                                     const float2* __restrict__ mlp, int64_t rows_heads, int32_t D,
                                                     float* __restrict__ O) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t rh = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; rh < rows_heads; rh += nw) {
        const float2 ml = lane < parts ? mlp[(int64_t)lane * rows_heads + rh] : make_float2(-INFINITY, 0.f);
        float M = ml.x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float wgt = lane < parts ? exp2f(ml.x - M) : 0.f;
        float l = 0.f;
        for (int g = 0; g < parts; ++g) l = fmaf(__shfl_sync(0xffffffffu, wgt, g), __shfl_sync(0xffffffffu, ml.y, g), l);
        const float inv = l > 0.f ? 1.f / l : 0.f;  // empty row -> 0 (reading c4)
        for (int f = lane; f < D; f += 32) {
            float acc = 0.f;
            for (int g = 0; g < parts; ++g)
                acc = fmaf(__shfl_sync(0xffffffffu, wgt, g), Op[((int64_t)g * rows_heads + rh) * D + f], acc);
            O[rh * D + f] = acc * inv;
        }
    }
}

// ---- host side ------------------------------------------------------------------------------------
// tensor-map helpers (also used by backward_sm100.cu; declared in internal.h)
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

// 2-D tensor map over a row-major [rows, inner] matrix; 16-bit elements use 64-element (128-byte)
// boxes with the 128-byte swizzle of the UMMA tiles, fp32 (O) a dense unswizzled box_inner-wide box
// Encoding a tensor map costs a few microseconds of host time per call, which dominates small
// launches (cora); the last few encodings are reused (per host thread) for identical arguments.
struct MapKey {
    const void* base;
    int64_t inner, rows, ld;
    uint32_t type, box_inner, box_rows, swz;
    bool operator==(const MapKey& o) const {
        return base == o.base && inner == o.inner && rows == o.rows && ld == o.ld && type == o.type &&
               box_inner == o.box_inner && box_rows == o.box_rows && swz == o.swz;
    }
};
f3s_status make_map_uncached(CUtensorMap* map, const void* base, CUtensorMapDataType type, int64_t inner,
                             int64_t rows, int64_t ld, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz);
// ld: elements between consecutive rows (>= inner)
f3s_status make_map(CUtensorMap* map, const void* base, CUtensorMapDataType type, int64_t inner, int64_t rows,
                    int64_t ld, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz) {
    constexpr int kCache = 8;
    thread_local MapKey keys[kCache];
    thread_local CUtensorMap maps[kCache];
    thread_local int used = 0, next = 0;
    const MapKey k{base, inner, rows, ld, (uint32_t)type, box_inner, box_rows, (uint32_t)swz};
    for (int i = 0; i < used; ++i)
        if (keys[i] == k) {
            *map = maps[i];
            return F3S_OK;
        }
    f3s_status st = make_map_uncached(map, base, type, inner, rows, ld, box_inner, box_rows, swz);
    if (st != F3S_OK) return st;
    keys[next] = k;
    maps[next] = *map;
    next = (next + 1) % kCache;
    if (used < kCache) ++used;
    return F3S_OK;
}
f3s_status make_map_uncached(CUtensorMap* map, const void* base, CUtensorMapDataType type, int64_t inner,
                             int64_t rows, int64_t ld, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz) {
    EncodeTiledFn enc = get_encode();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return F3S_ERR_CUDA; }
    const int esz = type == CU_TENSOR_MAP_DATA_TYPE_FLOAT32 ? 4 : type == CU_TENSOR_MAP_DATA_TYPE_UINT8 ? 1 : 2;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, type, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
        return F3S_ERR_CUDA;
    }
    return F3S_OK;
}
f3s_status make_map(CUtensorMap* map, const void* base, f3s_dtype dtype, int64_t inner, int64_t rows, int64_t ld,
                    uint32_t box_rows) {
    if (dtype == F3S_E4M3)  // 8-bit elements: 128-element (128-byte) boxes
        return make_map(map, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, inner, rows, ld, 128, box_rows,
                        CU_TENSOR_MAP_SWIZZLE_128B);
    return make_map(map, base, dtype == F3S_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                    inner, rows, ld, 64, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}


namespace {

template <int D, typename T, int HG>
f3s_status launch(const AttnArgs& a) {
    using C = Cfg<D, HG, (int)sizeof(T)>;
    const Plan& p = *a.plan;
    const int64_t out_bytes = (int64_t)p.n_rows * a.heads * D * 4;
    if (p.nnz == 0 || p.n_cols == 0) {  // every row is empty: O = 0 (reading c4)
        F3S_CUDA_TRY(cudaMemsetAsync(a.O, 0, (size_t)out_bytes, a.stream));
        return F3S_OK;
    }
    CUtensorMap mq, mo;
    f3s_status st;
    if ((st = make_map(&mq, a.Q, a.dtype, (int64_t)a.heads * D, p.n_rows, a.q_ld > 0 ? a.q_ld : (int64_t)a.heads * D,
                       16)) != F3S_OK)
        return st;
    if ((st = make_map(&mo, a.O, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (int64_t)a.heads * D, p.n_rows, (int64_t)a.heads * D,
                       D * HG, 16,
                       CU_TENSOR_MAP_SWIZZLE_NONE)) != F3S_OK)
        return st;

    // per-device launch state: SM count and the raised dynamic shared-memory limit (a function
    // attribute is per device, so it is set once on every device the library launches on)
    static std::atomic<int> num_sms[64];
    static std::atomic<uint64_t> attr_set{0};
    static std::mutex attr_mu;
    const int dev = p.device;
    if (dev < 0 || dev >= 64) { set_error("device ordinal >= 64"); return F3S_ERR_UNSUPPORTED; }
    if (!(attr_set.load() >> dev & 1)) {
        std::lock_guard<std::mutex> lock(attr_mu);
        if (!(attr_set.load() >> dev & 1)) {
            int v = 0;
            F3S_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
            num_sms[dev].store(v);
            F3S_CUDA_TRY(cudaFuncSetAttribute(k_f3s_sm100<D, T, false, HG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              C::kSmemBytes));
            F3S_CUDA_TRY(cudaFuncSetAttribute(k_f3s_sm100<D, T, true, HG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              C::kSmemBytes));
            if (HG > 1)
                F3S_CUDA_TRY(cudaFuncSetAttribute(k_f3s_sm100<D, T, false, HG, true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
            attr_set.fetch_or(uint64_t(1) << dev);
        }
    }
    const int sms = num_sms[dev].load();
    // default variant: the LPT list with heavy row windows split into pieces (Plan::meta_sub)
    const bool split = a.lpt && p.n_groups > 0 && a.sub_begin == 0;  // pieces lead the LPT list
    if (split && HG > 1) { set_error("internal: head groups with split windows"); return F3S_ERR_INTERNAL; }
    const int32_t sub_end = a.sub_end < 0 ? p.n_sub : a.sub_end;
    const int64_t n_items64 = (int64_t)(a.lpt ? sub_end - a.sub_begin : p.num_rw) * (a.heads / HG);
    if (n_items64 > 0x7FFFFFFF) { set_error("too many work items"); return F3S_ERR_UNSUPPORTED; }
    const int32_t n_items = (int32_t)n_items64;
    int64_t ctas = (int64_t)sms * C::kCtasPerSm;
    if (a.max_ctas > 0) ctas = std::min<int64_t>(ctas, a.max_ctas);  // SMs left free for a concurrent collective
    const int grid = a.grid_override > 0 ? a.grid_override : (int)std::min<int64_t>(n_items, ctas);
    // per-call scratch, stream-ordered (so calls in flight on other streams, or replays of a
    // captured graph, never share it): the work-queue counter, then for split plans one
    // (m[16], l[16], O[16][D]) fp32 record per piece and head
    const size_t rec_bytes = split ? sizeof(float) * (size_t)p.n_pieces * a.heads * (32 + 16 * D) : 0;
    char* scratch = nullptr;
    F3S_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&scratch), 256 + rec_bytes, a.stream));
    int32_t* counter = reinterpret_cast<int32_t*>(scratch);
    cudaError_t err = cudaMemsetAsync(counter, 0, sizeof(int32_t), a.stream);
    if (err == cudaSuccess) {
        auto kern = (a.trace || a.expt) ? k_f3s_sm100<D, T, true, HG>
                    : (HG > 1 && a.ml_out) ? k_f3s_sm100<D, T, false, HG, true> : k_f3s_sm100<D, T, false, HG>;
        kern<<<grid, C::kThreads, C::kSmemBytes, a.stream>>>(
            mq, mo, a.lpt ? p.meta_sub + a.sub_begin : p.meta_nat, p.kcols, p.kmasks, counter, n_items, a.heads,
            (a.kv_ld > 0 ? a.kv_ld : (int64_t)a.heads * D) * (int64_t)sizeof(T),
            static_cast<const uint8_t*>(a.K), static_cast<const uint8_t*>(a.V), a.scale * 1.4426950408889634f, a.trace,
            a.trace_chunks, a.expt, split ? reinterpret_cast<float*>(scratch + 256) : nullptr,
            reinterpret_cast<float2*>(a.ml_out), p.n_rows, a.O,
            a.lpt ? (int32_t)std::min<int64_t>((int64_t)std::max(0, p.n_heavy_sub - a.sub_begin) * (a.heads / HG),
                                               0x7FFFFFFF)
                  : 0,
            a.ml_norm ? 1 : 0);
        count_launch();
        err = cudaGetLastError();
    }
    if (err == cudaSuccess && split) {
        k_split_merge<D><<<(int)((int64_t)p.n_groups * a.heads), 256, 0, a.stream>>>(
            p.ginfo, reinterpret_cast<const float*>(scratch + 256), a.O, a.heads, p.n_rows,
            reinterpret_cast<float2*>(a.ml_out), a.ml_norm ? 1 : 0);
        count_launch();
        err = cudaGetLastError();
    }
    const cudaError_t ferr = scratch_free(scratch, a.stream);
    F3S_CUDA_TRY(err);
    F3S_CUDA_TRY(ferr);
    return F3S_OK;
}

}  // namespace

f3s_status launch_attention_sm100(const AttnArgs& a) {
    const Plan& p = *a.plan;
    if (a.dtype == F3S_E4M3) {
        // d = 64: the Q box (128 elements) also covers the next head's 64 (zero-filled past the
        // last head by the tensor map); MMA1 reads only the first 64 bytes of each row
        return a.d == 128 ? launch<128, __nv_fp8_e4m3, 1>(a) : launch<64, __nv_fp8_e4m3, 1>(a);
    }
    // head groups of 4 for row windows of at most 32 columns (d = 64): the per-chunk pipeline cost
    // is shared by 4 heads (batched small graphs).  In LPT order those windows form the tail of the
    // work list, so a plan with both kinds runs the wide head (and every split piece) one head per
    // chunk, then the narrow tail with head groups: two launches, the same per-head arithmetic
    // (reading c22)
    const bool hg_ok = !a.one_head && a.d == 64 && a.heads % 4 == 0 && p.nnz > 0 && p.n_cols > 0;
    if (hg_ok && a.lpt && a.sub_end < 0 && p.n_wide_sub > 0 && p.n_wide_sub < p.n_sub) {
        AttnArgs wide = a, narrow = a;
        wide.sub_begin = 0;
        wide.sub_end = p.n_wide_sub;
        narrow.sub_begin = p.n_wide_sub;
        narrow.sub_end = p.n_sub;
        f3s_status st = a.dtype == F3S_FP16 ? launch<64, __half, 1>(wide) : launch<64, __nv_bfloat16, 1>(wide);
        if (st != F3S_OK) return st;
        return a.dtype == F3S_FP16 ? launch<64, __half, 4>(narrow) : launch<64, __nv_bfloat16, 4>(narrow);
    }
    const bool hg4 = hg_ok && p.max_width <= 32 && p.n_groups == 0;
    if (a.dtype == F3S_FP16) {
        if (hg4) return launch<64, __half, 4>(a);
        return a.d == 64 ? launch<64, __half, 1>(a) : launch<128, __half, 1>(a);
    }
    if (hg4) return launch<64, __nv_bfloat16, 4>(a);
    return a.d == 64 ? launch<64, __nv_bfloat16, 1>(a) : launch<128, __nv_bfloat16, 1>(a);
}

__global__ void k_fill_ml(float2* __restrict__ ml, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ml[i] = make_float2(kMFloor, 0.f);
}

f3s_status launch_fill_ml(float* ml, int64_t rows_heads, cudaStream_t stream) {
    if (rows_heads == 0) return F3S_OK;
    k_fill_ml<<<(int)std::min<int64_t>((rows_heads + 255) / 256, 148 * 8), 256, 0, stream>>>(
        reinterpret_cast<float2*>(ml), rows_heads);
    count_launch();
    F3S_CUDA_TRY(cudaGetLastError());
    return F3S_OK;
}

f3s_status launch_parts_merge(int32_t parts, const float* O_parts, const float* ml_parts, int64_t rows_heads, int32_t d,
                              float* O, cudaStream_t stream) {
    if (rows_heads == 0) return F3S_OK;
    const int64_t blocks = std::min<int64_t>((rows_heads + 7) / 8, 148 * 16);
    k_parts_merge<<<(int)blocks, 256, 0, stream>>>(parts, O_parts, reinterpret_cast<const float2*>(ml_parts), rows_heads,
                                                   d, O);
    count_launch();
    F3S_CUDA_TRY(cudaGetLastError());
    return F3S_OK;
}

}  // namespace f3s
