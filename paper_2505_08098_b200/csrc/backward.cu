// backward.cu — gradients of the fused 3S pass ("the backward
// pass ... involves SpMM and SDDMM operations in reverse order").
//
// For O = softmax_row(scale * (Q K^T) (.) A) V (Eq.1) and dO = dL/dO:
//   dp_ij = dO_i . v_j,  D_i = sum_j p_ij dp_ij,  ds_ij = p_ij (dp_ij - D_i)
//   dQ_i = scale sum_j ds_ij k_j,  dK_j = scale sum_i ds_ij q_i,  dV_j = sum_i p_ij dO_i.
// Two deterministic passes, no atomics on the data:
//   row pass    one warp per (query row, head) (8 warps for rows of > 256 entries), walking its
//               row window's compacted columns
//               with the row's mask bit (the forward's plan): online max / sum / D (the same
//               rescaling as Alg.1 l.16-18), then p, ds and dQ; it leaves LSE_i and D_i.
//   column pass one warp per (key column, head) (8 for > 64 rows), walking the column's rows of A^T in ascending
//               order (a transposed index built once per plan from the plan's masks): it
//               recomputes p_ij = 2^(s_ij - LSE_i) and ds_ij and accumulates dK_j, dV_j.
// CUDA-core kernels (first version of the NEXT row f3): the tensor-core form would reuse the
// forward's chunk pipeline with the roles of the operands exchanged.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cub/cub.cuh>

#include <vector>

#include "internal.h"

namespace f3s {
namespace {

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---- row pass: dQ, LSE, D -------------------------------------------------------------------
template <int D, typename T>
__global__ void __launch_bounds__(512) k_bwd_rows(const int32_t* __restrict__ rw_ptr, const int32_t* __restrict__ cols,
                                                  const uint16_t* __restrict__ masks, int32_t n_rows, int H,
                                                  const T* __restrict__ Q, const T* __restrict__ K,
                                                  const T* __restrict__ V, const float* __restrict__ dO,
                                                  float* __restrict__ dQ, float* __restrict__ lse,
                                                  float* __restrict__ Drow, float scale,
                                                  const uint8_t* __restrict__ heavy_row) {
    constexpr int E = D / 32;  // features per lane
    const float scale_log2 = scale * 1.4426950408889634f;
    const int k = blockIdx.x / H, h = blockIdx.x - (blockIdx.x / H) * H;
    const int i = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = 16 * (int64_t)k + i;
    if (row >= n_rows || heavy_row[row]) return;  // heavy rows: k_bwd_rows_heavy
    const int64_t ld = (int64_t)H * D, base = row * ld + h * D + lane * E;
    float q[E], g[E], acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { q[e] = to_f(Q[base + e]); g[e] = dO[base + e]; acc[e] = 0.f; }
    const int32_t b = rw_ptr[k], en = rw_ptr[k + 1];
    // the row's entries among the window's compacted columns, 32 at a time: lane t tests entry
    // p0 + t, a ballot lists the hits, the warp walks the set bits
#define F3S_FOR_ROW_ENTRIES(...)                                                               \
    for (int32_t p0 = b; p0 < en; p0 += 32) {                                                  \
        const int32_t pl = p0 + lane;                                                          \
        uint32_t hits = __ballot_sync(0xffffffffu, pl < en && ((masks[pl] >> i) & 1));         \
        const int32_t cl = pl < en ? cols[pl] : 0;                                             \
        while (hits) {                                                                         \
            const int t = __ffs(hits) - 1;                                                     \
            hits &= hits - 1;                                                                  \
            const int64_t jb = (int64_t)__shfl_sync(0xffffffffu, cl, t) * ld + h * D + lane * E; \
            __VA_ARGS__                                                                        \
        }                                                                                      \
    }
    // pass 1: running max m (log2 units), l = sum 2^(x - m), u = sum 2^(x - m) dp  -> D = u / l
    float m = -INFINITY, l = 0.f, u = 0.f;
    F3S_FOR_ROW_ENTRIES({
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) { s += q[e] * to_f(K[jb + e]); dp += g[e] * to_f(V[jb + e]); }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float x = s * scale_log2;
        const float mn = fmaxf(m, x);
        const float a = exp2f(m - mn), w = exp2f(x - mn);  // m = -inf at the first entry -> a = 0
        l = l * a + w;
        u = u * a + w * dp;
        m = mn;
    })
    const float L = m + log2f(l);  // row log-sum-exp in log2 units (-inf for an empty row)
    const float Di = l > 0.f ? u / l : 0.f;
    // pass 2: p = 2^(x - L), ds = p (dp - D), dQ += scale ds k
    F3S_FOR_ROW_ENTRIES({
        float kv[E], s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) { kv[e] = to_f(K[jb + e]); s += q[e] * kv[e]; dp += g[e] * to_f(V[jb + e]); }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float ds = exp2f(s * scale_log2 - L) * (dp - Di);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = fmaf(scale * ds, kv[e], acc[e]);
    })
#undef F3S_FOR_ROW_ENTRIES
#pragma unroll
    for (int e = 0; e < E; ++e) dQ[base + e] = acc[e];  // empty row: 0
    if (lane == 0) {
        lse[row * H + h] = L;
        Drow[row * H + h] = Di;
    }
}

// heavy rows (more than kHeavyRow entries): one block of 8 warps per (row, head); warp w walks
// the window entry blocks w, w+8, ... ; the per-warp (max, sum, D-sum) and dQ partials are
// combined in warp order (deterministic)
constexpr int kHeavyRow = 256;
template <int D, typename T>
__global__ void __launch_bounds__(256) k_bwd_rows_heavy(const int32_t* __restrict__ heavy, const int32_t* __restrict__ rw_ptr,
                                                        const int32_t* __restrict__ cols, const uint16_t* __restrict__ masks,
                                                        int H, const T* __restrict__ Q, const T* __restrict__ K,
                                                        const T* __restrict__ V, const float* __restrict__ dO,
                                                        float* __restrict__ dQ, float* __restrict__ lse,
                                                        float* __restrict__ Drow, float scale) {
    constexpr int E = D / 32;
    __shared__ float st[8][3];
    __shared__ float part[8][D];
    const float scale_log2 = scale * 1.4426950408889634f;
    const int64_t row = heavy[blockIdx.x / H];
    const int h = blockIdx.x - (blockIdx.x / H) * H;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = (int)(row & 15);
    const int64_t k = row >> 4;
    const int64_t ld = (int64_t)H * D, base = row * ld + h * D + lane * E;
    float q[E], g[E], acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { q[e] = to_f(Q[base + e]); g[e] = dO[base + e]; acc[e] = 0.f; }
    const int32_t b = rw_ptr[k], en = rw_ptr[k + 1];
#define F3S_FOR_MY_ENTRIES(...)                                                                \
    for (int32_t p0 = b + 32 * w; p0 < en; p0 += 256) {                                        \
        const int32_t pl = p0 + lane;                                                          \
        uint32_t hits = __ballot_sync(0xffffffffu, pl < en && ((masks[pl] >> i) & 1));         \
        const int32_t cl = pl < en ? cols[pl] : 0;                                             \
        while (hits) {                                                                         \
            const int t = __ffs(hits) - 1;                                                     \
            hits &= hits - 1;                                                                  \
            const int64_t jb = (int64_t)__shfl_sync(0xffffffffu, cl, t) * ld + h * D + lane * E; \
            __VA_ARGS__                                                                        \
        }                                                                                      \
    }
    float m = -INFINITY, l = 0.f, u = 0.f;
    F3S_FOR_MY_ENTRIES({
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) { s += q[e] * to_f(K[jb + e]); dp += g[e] * to_f(V[jb + e]); }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float x = s * scale_log2;
        const float mn = fmaxf(m, x);
        const float a = exp2f(m - mn), wt = exp2f(x - mn);
        l = l * a + wt;
        u = u * a + wt * dp;
        m = mn;
    })
    if (lane == 0) { st[w][0] = m; st[w][1] = l; st[w][2] = u; }
    __syncthreads();
    float M = -INFINITY;
#pragma unroll
    for (int v = 0; v < 8; ++v) M = fmaxf(M, st[v][0]);
    float lt = 0.f, ut = 0.f;
#pragma unroll
    for (int v = 0; v < 8; ++v) {  // warps without entries have l = u = 0 (m = -inf -> weight 0)
        const float sc = st[v][1] > 0.f ? exp2f(st[v][0] - M) : 0.f;
        lt = fmaf(st[v][1], sc, lt);
        ut = fmaf(st[v][2], sc, ut);
    }
    const float L = M + log2f(lt), Di = lt > 0.f ? ut / lt : 0.f;
    F3S_FOR_MY_ENTRIES({
        float kv[E], s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) { kv[e] = to_f(K[jb + e]); s += q[e] * kv[e]; dp += g[e] * to_f(V[jb + e]); }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float ds = exp2f(s * scale_log2 - L) * (dp - Di);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = fmaf(scale * ds, kv[e], acc[e]);
    })
#undef F3S_FOR_MY_ENTRIES
#pragma unroll
    for (int e = 0; e < E; ++e) part[w][lane * E + e] = acc[e];
    __syncthreads();
    for (int f = threadIdx.x; f < D; f += blockDim.x) {
        float a2 = 0.f;
#pragma unroll
        for (int v = 0; v < 8; ++v) a2 += part[v][f];  // fixed order
        dQ[row * ld + h * D + f] = a2;
    }
    if (threadIdx.x == 0) {
        lse[row * H + h] = L;
        Drow[row * H + h] = Di;
    }
}

// per-row entry counts from the plan's masks (row degrees of the deduplicated A)
__global__ void k_row_deg(const int32_t* __restrict__ rw_ptr, int32_t R, const uint16_t* __restrict__ masks,
                          int32_t* __restrict__ deg) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)R * 16;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t >> 4;
        const int i = (int)(t & 15);
        int32_t c = 0;
        for (int32_t p = rw_ptr[k]; p < rw_ptr[k + 1]; ++p) c += (masks[p] >> i) & 1;
        deg[t] = c;
    }
}

// ---- column pass: dK, dV -------------------------------------------------------------------
template <int D, typename T>
__global__ void __launch_bounds__(256) k_bwd_cols(const int32_t* __restrict__ light, const int32_t* __restrict__ col_ptr,
                                                  const int32_t* __restrict__ col_rows, int32_t n_cols, int H,
                                                  const T* __restrict__ Q,
                                                  const T* __restrict__ K, const T* __restrict__ V,
                                                  const float* __restrict__ dO, const float* __restrict__ lse,
                                                  const float* __restrict__ Drow, float* __restrict__ dK,
                                                  float* __restrict__ dV, float scale) {
    constexpr int E = D / 32;
    const float scale_log2 = scale * 1.4426950408889634f;
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (wid >= (int64_t)n_cols * H) return;  // n_cols: number of light columns
    const int64_t j = light[wid / H];
    const int h = (int)(wid - (wid / H) * H);
    const int64_t ld = (int64_t)H * D, jb = j * ld + h * D + lane * E;
    float kv[E], vv[E], gk[E], gv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { kv[e] = to_f(K[jb + e]); vv[e] = to_f(V[jb + e]); gk[e] = 0.f; gv[e] = 0.f; }
    for (int32_t t = col_ptr[j]; t < col_ptr[j + 1]; ++t) {
        const int64_t i = col_rows[t];
        const int64_t ib = i * ld + h * D + lane * E;
        float qv[E], gi[E], s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            qv[e] = to_f(Q[ib + e]);
            gi[e] = dO[ib + e];
            s += qv[e] * kv[e];
            dp += gi[e] * vv[e];
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float pij = exp2f(s * scale_log2 - lse[i * H + h]);
        const float ds = pij * (dp - Drow[i * H + h]);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            gk[e] = fmaf(scale * ds, qv[e], gk[e]);
            gv[e] = fmaf(pij, gi[e], gv[e]);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) { dK[jb + e] = gk[e]; dV[jb + e] = gv[e]; }
}

// heavy columns (more than kHeavyCol rows: power-law in-degree hubs): one block of NW = 8 (32 above
// kHugeCol rows) warps per (column, head); warp w takes rows w, w+NW, ... and the NW partial sums
// are added in warp order
// (deterministic).  A hub of 13,000 rows on one warp alone set the whole pass's time.
constexpr int kHeavyCol = 64, kHugeCol = 1024;  // > kHugeCol rows: 32 warps
template <int D, typename T, int NW>
__global__ void __launch_bounds__(32 * NW) k_bwd_cols_heavy(const int32_t* __restrict__ heavy, const int32_t* __restrict__ col_ptr,
                                                        const int32_t* __restrict__ col_rows, int H,
                                                        const T* __restrict__ Q, const T* __restrict__ K,
                                                        const T* __restrict__ V, const float* __restrict__ dO,
                                                        const float* __restrict__ lse, const float* __restrict__ Drow,
                                                        float* __restrict__ dK, float* __restrict__ dV, float scale) {
    constexpr int E = D / 32;
    __shared__ float part[NW][2][D];
    const float scale_log2 = scale * 1.4426950408889634f;
    const int64_t j = heavy[blockIdx.x / H];
    const int h = blockIdx.x - (blockIdx.x / H) * H;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ld = (int64_t)H * D, jb = j * ld + h * D + lane * E;
    float kv[E], vv[E], gk[E], gv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { kv[e] = to_f(K[jb + e]); vv[e] = to_f(V[jb + e]); gk[e] = 0.f; gv[e] = 0.f; }
    for (int32_t t = col_ptr[j] + w; t < col_ptr[j + 1]; t += NW) {
        const int64_t i = col_rows[t];
        const int64_t ib = i * ld + h * D + lane * E;
        float qv[E], gi[E], s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            qv[e] = to_f(Q[ib + e]);
            gi[e] = dO[ib + e];
            s += qv[e] * kv[e];
            dp += gi[e] * vv[e];
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float pij = exp2f(s * scale_log2 - lse[i * H + h]);
        const float ds = pij * (dp - Drow[i * H + h]);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            gk[e] = fmaf(scale * ds, qv[e], gk[e]);
            gv[e] = fmaf(pij, gi[e], gv[e]);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) { part[w][0][lane * E + e] = gk[e]; part[w][1][lane * E + e] = gv[e]; }
    __syncthreads();
    for (int f = threadIdx.x; f < 2 * D; f += blockDim.x) {
        const int which = f / D, x = f - which * D;
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < NW; ++u) acc += part[u][which][x];  // fixed order
        (which ? dV : dK)[j * ld + h * D + x] = acc;
    }
}

// ---- transposed index of A (built once per plan) ----------------------------------------------
// per plan entry (compacted column of a window): the popcount of its mask (rows in A^T)
__global__ void k_entry_pop(const int32_t* __restrict__ cols, const uint16_t* __restrict__ masks, int64_t W,
                            int32_t* __restrict__ pop, int32_t* __restrict__ col_cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < W; p += (int64_t)gridDim.x * blockDim.x) {
        const int c = __popc((uint32_t)masks[p]);
        pop[p] = c;
        if (c) atomicAdd(&col_cnt[cols[p]], c);
    }
}
// the window of each entry is found from rw_ptr by the writer: one warp per window
__global__ void k_entry_keys(const int32_t* __restrict__ rw_ptr, int32_t R, const int32_t* __restrict__ cols,
                             const uint16_t* __restrict__ masks, const int32_t* __restrict__ off,
                             uint64_t* __restrict__ keys) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < R; k += nw)
        for (int32_t p = rw_ptr[k] + lane; p < rw_ptr[k + 1]; p += 32) {
            uint32_t mk = masks[p];
            int32_t o = off[p];
            while (mk) {
                const int i = __ffs(mk) - 1;
                mk &= mk - 1;
                keys[o++] = ((uint64_t)(uint32_t)cols[p] << 32) | (uint64_t)(16 * k + i);
            }
        }
}
__global__ void k_key_rows(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ rows) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        rows[t] = (int32_t)(keys[t] & 0xFFFFFFFFu);
}

int grid_for(int64_t n, int block) {
    const int64_t g = (n + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() { if (p) scratch_free(p, s); }
};

f3s_status build_transpose(Plan& p, cudaStream_t stream) {
    std::lock_guard<std::mutex> lock(p.transpose_mu);  // concurrent first backward calls build it once
    if (p.col_ptr) return F3S_OK;
    const int64_t W = p.total_cols, nnz = p.nnz;
    int32_t *col_ptr = nullptr, *col_rows = nullptr;
    F3S_CUDA_TRY(cudaMalloc(&col_ptr, sizeof(int32_t) * ((size_t)p.n_cols + 1)));
    F3S_CUDA_TRY(cudaMalloc(&col_rows, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1)));
    Scratch pop, off, cnt, keys, keys2, tmp;
    pop.s = off.s = cnt.s = keys.s = keys2.s = tmp.s = stream;
    F3S_CUDA_TRY(scratch_alloc(&pop.p, sizeof(int32_t) * (size_t)std::max<int64_t>(W, 1), stream));
    F3S_CUDA_TRY(scratch_alloc(&off.p, sizeof(int32_t) * (size_t)std::max<int64_t>(W, 1), stream));
    F3S_CUDA_TRY(scratch_alloc(&cnt.p, sizeof(int32_t) * ((size_t)p.n_cols + 1), stream));
    F3S_CUDA_TRY(scratch_alloc(&keys.p, sizeof(uint64_t) * (size_t)std::max<int64_t>(nnz, 1), stream));
    F3S_CUDA_TRY(scratch_alloc(&keys2.p, sizeof(uint64_t) * (size_t)std::max<int64_t>(nnz, 1), stream));
    F3S_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(int32_t) * ((size_t)p.n_cols + 1), stream));
    if (W > 0) {
        k_entry_pop<<<grid_for(W, 256), 256, 0, stream>>>(p.cols, p.masks, W, (int32_t*)pop.p, (int32_t*)cnt.p);
        count_launch();
    }
    size_t tb_scan = 0, tb_scan2 = 0, tb_sort = 0;
    F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, (int32_t*)pop.p, (int32_t*)off.p, W, stream));
    F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb_scan2, (int32_t*)cnt.p, col_ptr, (int64_t)p.n_cols + 1, stream));
    cub::DoubleBuffer<uint64_t> db((uint64_t*)keys.p, (uint64_t*)keys2.p);
    F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, db, nnz, 0, 64, stream));
    F3S_CUDA_TRY(scratch_alloc(&tmp.p, std::max(std::max(tb_scan, tb_scan2), tb_sort) + 16, stream));
    const size_t tbmax = std::max(std::max(tb_scan, tb_scan2), tb_sort) + 16;
    size_t tb = tbmax;
    if (W > 0) F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)pop.p, (int32_t*)off.p, W, stream));
    tb = tbmax;
    F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, tb, (int32_t*)cnt.p, col_ptr, (int64_t)p.n_cols + 1, stream));
    count_launch(2);
    if (nnz > 0) {
        k_entry_keys<<<grid_for((int64_t)p.num_rw * 32, 256), 256, 0, stream>>>(p.rw_ptr, p.num_rw, p.cols, p.masks,
                                                                               (int32_t*)off.p, (uint64_t*)keys.p);
        count_launch();
        tb = tbmax;
        F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, nnz, 0, 64, stream));  // (column, row) ascending
        count_launch();
        k_key_rows<<<grid_for(nnz, 256), 256, 0, stream>>>(db.Current(), nnz, col_rows);
        count_launch();
    }
    F3S_CUDA_TRY(cudaGetLastError());
    // light / heavy column lists (one-time host pass over the column counts)
    std::vector<int32_t> h_cp((size_t)p.n_cols + 1);
    F3S_CUDA_TRY(cudaMemcpyAsync(h_cp.data(), col_ptr, sizeof(int32_t) * h_cp.size(), cudaMemcpyDeviceToHost, stream));
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    std::vector<int32_t> light, heavy, huge;
    for (int32_t j = 0; j < p.n_cols; ++j) {
        const int32_t c = h_cp[j + 1] - h_cp[j];
        if (c > kHugeCol) huge.push_back(j);
        else if (c > kHeavyCol) heavy.push_back(j);
        else if (c > 0) light.push_back(j);
    }
    const int32_t n_heavy8 = (int32_t)heavy.size();
    heavy.insert(heavy.end(), huge.begin(), huge.end());  // heavy list: 8-warp columns, then 32-warp ones
    // (columns without rows get dK = dV = 0 from a memset in launch_bwd)
    int32_t* lists = nullptr;
    F3S_CUDA_TRY(cudaMalloc(&lists, sizeof(int32_t) * (light.size() + heavy.size() + 1)));
    if (!light.empty())
        F3S_CUDA_TRY(cudaMemcpy(lists, light.data(), sizeof(int32_t) * light.size(), cudaMemcpyHostToDevice));
    if (!heavy.empty())
        F3S_CUDA_TRY(cudaMemcpy(lists + light.size(), heavy.data(), sizeof(int32_t) * heavy.size(), cudaMemcpyHostToDevice));
    // heavy rows: degree from the plan's masks
    std::vector<int32_t> h_deg((size_t)p.num_rw * 16);
    {
        Scratch degs;
        degs.s = stream;
        F3S_CUDA_TRY(scratch_alloc(&degs.p, sizeof(int32_t) * h_deg.size() + 16, stream));
        k_row_deg<<<grid_for((int64_t)p.num_rw * 16, 256), 256, 0, stream>>>(p.rw_ptr, p.num_rw, p.masks,
                                                                             (int32_t*)degs.p);
        count_launch();
        F3S_CUDA_TRY(cudaMemcpyAsync(h_deg.data(), degs.p, sizeof(int32_t) * h_deg.size(), cudaMemcpyDeviceToHost,
                                     stream));
        F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    }
    std::vector<int32_t> hrows;
    std::vector<uint8_t> flag((size_t)std::max(p.n_rows, 1), 0);
    for (int32_t r = 0; r < p.n_rows; ++r)
        if (h_deg[r] > kHeavyRow) { hrows.push_back(r); flag[r] = 1; }
    int32_t* hr = nullptr;
    uint8_t* hf = nullptr;
    F3S_CUDA_TRY(cudaMalloc(&hr, sizeof(int32_t) * (hrows.size() + 1)));
    F3S_CUDA_TRY(cudaMalloc(&hf, flag.size()));
    if (!hrows.empty()) F3S_CUDA_TRY(cudaMemcpy(hr, hrows.data(), sizeof(int32_t) * hrows.size(), cudaMemcpyHostToDevice));
    F3S_CUDA_TRY(cudaMemcpy(hf, flag.data(), flag.size(), cudaMemcpyHostToDevice));
    p.heavy_rows = hr;
    p.heavy_row_flag = hf;
    p.n_heavy_rows = (int32_t)hrows.size();
    p.col_ptr = col_ptr;
    p.col_rows = col_rows;
    p.col_lists = lists;
    p.n_light = (int32_t)light.size();
    p.n_heavy = (int32_t)heavy.size();
    p.n_heavy8 = n_heavy8;
    return F3S_OK;
}

template <int D, typename T>
f3s_status launch_bwd(Plan& p, const void* Q, const void* K, const void* V, const float* dO, float* dQ, float* dK,
                      float* dV, float scale, int H, cudaStream_t stream) {
    if (p.n_rows == 0 || p.nnz == 0) {
        if (p.n_rows) F3S_CUDA_TRY(cudaMemsetAsync(dQ, 0, sizeof(float) * (size_t)p.n_rows * H * D, stream));
        if (p.n_cols) {
            F3S_CUDA_TRY(cudaMemsetAsync(dK, 0, sizeof(float) * (size_t)p.n_cols * H * D, stream));
            F3S_CUDA_TRY(cudaMemsetAsync(dV, 0, sizeof(float) * (size_t)p.n_cols * H * D, stream));
        }
        return F3S_OK;
    }
    f3s_status st = build_transpose(p, stream);
    if (st != F3S_OK) return st;
    Scratch stats;
    stats.s = stream;
    F3S_CUDA_TRY(scratch_alloc(&stats.p, sizeof(float) * 2 * (size_t)p.n_rows * H, stream));
    float* lse = (float*)stats.p;
    float* drow = lse + (size_t)p.n_rows * H;
    const int64_t blocks = (int64_t)p.num_rw * H;
    if (blocks > 0x7FFFFFFF) { set_error("too many row blocks"); return F3S_ERR_UNSUPPORTED; }
    k_bwd_rows<D, T><<<(unsigned)blocks, 512, 0, stream>>>(p.rw_ptr, p.cols, p.masks, p.n_rows, H,
                                                           static_cast<const T*>(Q), static_cast<const T*>(K),
                                                           static_cast<const T*>(V), dO, dQ, lse, drow, scale,
                                                           p.heavy_row_flag);
    count_launch();
    if (p.n_heavy_rows > 0) {
        if ((int64_t)p.n_heavy_rows * H > 0x7FFFFFFF) { set_error("too many heavy rows"); return F3S_ERR_UNSUPPORTED; }
        k_bwd_rows_heavy<D, T><<<(unsigned)((int64_t)p.n_heavy_rows * H), 256, 0, stream>>>(
            p.heavy_rows, p.rw_ptr, p.cols, p.masks, H, static_cast<const T*>(Q), static_cast<const T*>(K),
            static_cast<const T*>(V), dO, dQ, lse, drow, scale);
        count_launch();
    }
    F3S_CUDA_TRY(cudaGetLastError());
    if (p.n_light + p.n_heavy < p.n_cols) {  // columns without rows: zero gradients
        F3S_CUDA_TRY(cudaMemsetAsync(dK, 0, sizeof(float) * (size_t)p.n_cols * H * D, stream));
        F3S_CUDA_TRY(cudaMemsetAsync(dV, 0, sizeof(float) * (size_t)p.n_cols * H * D, stream));
    }
    const int64_t warps = (int64_t)p.n_light * H, cblocks = (warps + 7) / 8;
    if (cblocks > 0x7FFFFFFF || (int64_t)p.n_heavy * H > 0x7FFFFFFF) {
        set_error("too many column blocks");
        return F3S_ERR_UNSUPPORTED;
    }
    if (cblocks > 0) {
        k_bwd_cols<D, T><<<(unsigned)cblocks, 256, 0, stream>>>(p.col_lists, p.col_ptr, p.col_rows, p.n_light, H,
                                                                static_cast<const T*>(Q), static_cast<const T*>(K),
                                                                static_cast<const T*>(V), dO, lse, drow, dK, dV, scale);
        count_launch();
    }
    if (p.n_heavy8 > 0) {
        k_bwd_cols_heavy<D, T, 8><<<(unsigned)((int64_t)p.n_heavy8 * H), 256, 0, stream>>>(
            p.col_lists + p.n_light, p.col_ptr, p.col_rows, H, static_cast<const T*>(Q), static_cast<const T*>(K),
            static_cast<const T*>(V), dO, lse, drow, dK, dV, scale);
        count_launch();
    }
    if (p.n_heavy > p.n_heavy8) {
        k_bwd_cols_heavy<D, T, 32><<<(unsigned)((int64_t)(p.n_heavy - p.n_heavy8) * H), 1024, 0, stream>>>(
            p.col_lists + p.n_light + p.n_heavy8, p.col_ptr, p.col_rows, H, static_cast<const T*>(Q),
            static_cast<const T*>(K), static_cast<const T*>(V), dO, lse, drow, dK, dV, scale);
        count_launch();
    }
    F3S_CUDA_TRY(cudaGetLastError());
    return F3S_OK;
}

}  // namespace

// Plan of A^T (rows = columns of A, compacted columns = rows of A) for the tensor-core column
// pass: built once per plan from the transposed index, under the plan's transpose lock.
f3s_status build_transpose_plan(Plan& p, cudaStream_t stream) {
    f3s_status st = build_transpose(p, stream);
    if (st != F3S_OK) return st;
    std::lock_guard<std::mutex> lock(p.transpose_mu);
    if (p.tplan) return F3S_OK;
    Plan* tp = nullptr;
    const int32_t* col_idx = p.col_rows;
    st = build_plan(p.col_ptr, col_idx, p.n_cols, p.n_rows, true, stream, &tp);
    if (st != F3S_OK) return st;
    p.tplan = tp;
    return F3S_OK;
}

f3s_status launch_attention_backward(Plan& p, const void* Q, const void* K, const void* V, const float* dO, float* dQ,
                                     float* dK, float* dV, float scale, int heads, int d, f3s_dtype dtype,
                                     cudaStream_t stream) {
    if (dtype == F3S_FP16)
        return d == 64 ? launch_bwd<64, __half>(p, Q, K, V, dO, dQ, dK, dV, scale, heads, stream)
                       : launch_bwd<128, __half>(p, Q, K, V, dO, dQ, dK, dV, scale, heads, stream);
    return d == 64 ? launch_bwd<64, __nv_bfloat16>(p, Q, K, V, dO, dQ, dK, dV, scale, heads, stream)
                   : launch_bwd<128, __nv_bfloat16>(p, Q, K, V, dO, dQ, dK, dV, scale, heads, stream);
}

}  // namespace f3s
