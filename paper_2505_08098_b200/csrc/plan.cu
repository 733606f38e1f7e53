// plan.cu — device-side builder of the row-window plan (§3.1) and of the
// row-window reordering.
//
// One global radix sort of the keys (rw << (colbits+4) | col << 4 | row&15) groups every
// row window's entries by column; a head-flag scan deduplicates (rw, col) pairs (column
// compaction); each run of equal (rw, col) ORs its row bits into the column's 16-bit
// mask (bitmap).  Widths are counted per window and scanned into rw_ptr (tro).
// The LPT order sorts unique keys ((2^32-1 - ceil(w/8)) << 32 | k), i.e. TCB count
// descending, index ascending (reading c13).  All integer work: bit-exact and
// deterministic.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.h"

namespace f3s {
namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

int bits_for(int64_t max_value) {  // bits needed to hold values in [0, max_value]
    int b = 1;
    while (b < 63 && (int64_t(1) << b) <= max_value) ++b;
    return b;
}

__global__ void k_check_rowptr(const int32_t* __restrict__ rp, int32_t n_rows, int32_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x)
        if (rp[i + 1] < rp[i]) atomicOr(flag, 1);
}

// one warp per row: key = rw << (colbits + 4) | col << 4 | (row & 15)
__global__ void k_make_keys(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int32_t n_rows,
                            int32_t n_cols, int colbits, int32_t base, uint64_t* __restrict__ keys,
                            int32_t* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nwarps) {
        const int32_t b = rp[r], e = rp[r + 1];
        const uint64_t hi = ((uint64_t)(r >> 4) << (colbits + 4)) | (uint64_t)(r & 15);
        for (int32_t p = b + lane; p < e; p += 32) {
            int32_t c = ci[p];
            if (c < 0 || c >= n_cols) { atomicOr(flag, 2); c = 0; }
            keys[p - base] = hi | ((uint64_t)c << 4);
        }
    }
}

__global__ void k_heads(const uint64_t* __restrict__ keys, int64_t m, int32_t* __restrict__ head) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x)
        head[p] = (p == 0 || (keys[p] >> 4) != (keys[p - 1] >> 4)) ? 1 : 0;
}

__global__ void k_fill(const uint64_t* __restrict__ keys, const int32_t* __restrict__ pos, int64_t m, int colbits,
                       int32_t* __restrict__ cols, uint16_t* __restrict__ masks, int32_t* __restrict__ widths,
                       unsigned long long* __restrict__ popcount) {
    const uint64_t colmask = (uint64_t(1) << colbits) - 1;
    unsigned long long acc = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t rc = keys[p] >> 4;
        if (p > 0 && (keys[p - 1] >> 4) == rc) continue;  // not the head of its (rw, col) run
        uint32_t mask = 0;
        for (int64_t q = p; q < m && (keys[q] >> 4) == rc; ++q) mask |= 1u << (keys[q] & 15);
        const int32_t u = pos[p] - 1;
        cols[u] = (int32_t)(rc & colmask);
        masks[u] = (uint16_t)mask;
        atomicAdd(&widths[rc >> colbits], 1);
        acc += (unsigned long long)__popc(mask);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(popcount, acc);
}

__global__ void k_order_keys(const int32_t* __restrict__ rw_ptr, int32_t R, uint64_t* __restrict__ okeys,
                             int32_t* __restrict__ natural) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < R; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t tcb8 = (uint32_t)((rw_ptr[k + 1] - rw_ptr[k] + 7) >> 3);
        okeys[k] = ((uint64_t)(0xFFFFFFFFu - tcb8) << 32) | (uint64_t)k;
        natural[k] = (int32_t)k;
    }
}

__global__ void k_order_extract(const uint64_t* __restrict__ okeys, int32_t R, int32_t* __restrict__ order) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < R; k += (int64_t)gridDim.x * blockDim.x)
        order[k] = (int32_t)(okeys[k] & 0xFFFFFFFFu);
}

__global__ void k_width8(const int32_t* __restrict__ rw_ptr, int32_t R, int32_t* __restrict__ w8) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= R; k += (int64_t)gridDim.x * blockDim.x)
        w8[k] = k < R ? ((rw_ptr[k + 1] - rw_ptr[k] + 7) & ~7) : 0;
}

// kernel layout: one warp per row window copies its columns/masks to an 8-aligned start and
// pads to a multiple of 8 with the last column (mask 0); plus the per-window meta records.
__global__ void k_kernel_layout(const int32_t* __restrict__ rw_ptr, const int32_t* __restrict__ rw_ptr8,
                                const int32_t* __restrict__ cols, const uint16_t* __restrict__ masks,
                                const int32_t* __restrict__ order, int32_t R, int32_t* __restrict__ kcols,
                                uint16_t* __restrict__ kmasks, int4* __restrict__ meta_lpt, int4* __restrict__ meta_nat) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < R; k += nwarps) {
        const int32_t b = rw_ptr[k], w = rw_ptr[k + 1] - b, b8 = rw_ptr8[k], w8 = rw_ptr8[k + 1] - b8;
        for (int32_t p = lane; p < w8; p += 32) {
            kcols[b8 + p] = cols[b + min(p, w - 1)];
            kmasks[b8 + p] = p < w ? masks[b + p] : (uint16_t)0;
        }
        if (lane == 0) meta_nat[k] = make_int4((int)k, b8, w, 0);
        const int32_t ko = order[k];
        if (lane == 1) meta_lpt[k] = make_int4(ko, rw_ptr8[ko], rw_ptr[ko + 1] - rw_ptr[ko], 0);
    }
}

int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

}  // namespace

f3s_status build_plan(const int32_t* row_ptr, const int32_t* col_idx, int32_t n_rows, int32_t n_cols,
                      bool require_zero_base, cudaStream_t stream, Plan** out) {
    *out = nullptr;
    if (n_rows < 0 || n_cols < 0) { set_error("negative n_rows/n_cols"); return F3S_ERR_INVALID_VALUE; }
    if (!row_ptr) { set_error("row_ptr is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (n_rows > 0x7FFFFFFF - 16) { set_error("n_rows too large"); return F3S_ERR_UNSUPPORTED; }

    Plan* plan = new (std::nothrow) Plan();
    if (!plan) return F3S_ERR_OUT_OF_MEMORY;
    struct Guard { Plan*& p; bool ok = false; ~Guard() { if (!ok && p) {
        cudaFree(p->rw_ptr); cudaFree(p->cols); cudaFree(p->masks); cudaFree(p->rw_order);
        cudaFree(p->rw_natural); cudaFree(p->kcols); cudaFree(p->kmasks);
        cudaFree(p->meta_lpt); cudaFree(p->meta_nat); cudaFree(p->meta_sub); cudaFree(p->ginfo); cudaFree(p->col_ptr); cudaFree(p->col_rows); cudaFree(p->col_lists); cudaFree(p->heavy_rows); cudaFree(p->heavy_row_flag); delete p; p = nullptr; } } } guard{plan};
    F3S_CUDA_TRY(cudaGetDevice(&plan->device));
    const int32_t R = (n_rows + kRowsPerWindow - 1) / kRowsPerWindow;
    plan->n_rows = n_rows;
    plan->n_cols = n_cols;
    plan->num_rw = R;

    cudaEvent_t ev0, ev1;
    F3S_CUDA_TRY(cudaEventCreate(&ev0));
    F3S_CUDA_TRY(cudaEventCreate(&ev1));
    struct EvGuard { cudaEvent_t a, b; ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); } } evg{ev0, ev1};
    F3S_CUDA_TRY(cudaEventRecord(ev0, stream));

    DevBuf flag;  // [0]: error bits (int32), [2..3]: deduplicated nnz (u64)
    F3S_CUDA_TRY(flag.alloc(4 * sizeof(int32_t)));
    F3S_CUDA_TRY(cudaMemsetAsync(flag.p, 0, 4 * sizeof(int32_t), stream));
    unsigned long long* d_pop = reinterpret_cast<unsigned long long*>(flag.as<int32_t>() + 2);

    // ---- 1. validate row_ptr and learn nnz (sync #1) -------------------------------------
    int32_t ends[2] = {0, 0};
    if (n_rows > 0) {
        k_check_rowptr<<<grid_for(n_rows, 256), 256, 0, stream>>>(row_ptr, n_rows, flag.as<int32_t>());
        count_launch();
        F3S_CUDA_TRY(cudaGetLastError());
        F3S_CUDA_TRY(cudaMemcpyAsync(&ends[0], row_ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        F3S_CUDA_TRY(cudaMemcpyAsync(&ends[1], row_ptr + n_rows, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    }
    int32_t hflag = 0;
    F3S_CUDA_TRY(cudaMemcpyAsync(&hflag, flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    if (hflag & 1) { set_error("row_ptr is not non-decreasing"); return F3S_ERR_INVALID_CSR; }
    if (ends[0] < 0 || (require_zero_base && ends[0] != 0)) {
        set_error("row_ptr[0] = " + std::to_string(ends[0]) + (require_zero_base ? " (must be 0)" : " (negative)"));
        return F3S_ERR_INVALID_CSR;
    }
    const int64_t nnz = (int64_t)ends[1] - ends[0];
    if (nnz > 0 && !col_idx) { set_error("col_idx is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (nnz > 0 && n_cols == 0) { set_error("entries present but n_cols == 0"); return F3S_ERR_INVALID_CSR; }

    const int colbits = bits_for(std::max<int64_t>(n_cols - 1, 1));
    const int rwbits = bits_for(std::max<int64_t>(R - 1, 1));
    if (colbits + rwbits + 4 > 64) { set_error("key does not fit 64 bits"); return F3S_ERR_UNSUPPORTED; }
    const int key_bits = colbits + rwbits + 4;

    // ---- 2. keys, sort, dedup (sync #2 to size cols/masks) -------------------------------
    DevBuf keys, keys_alt, pos, temp, widths;
    int64_t W = 0;
    F3S_CUDA_TRY(widths.alloc(sizeof(int32_t) * (size_t)(R + 1)));
    F3S_CUDA_TRY(cudaMemsetAsync(widths.p, 0, sizeof(int32_t) * (size_t)(R + 1), stream));
    if (nnz > 0) {
        F3S_CUDA_TRY(keys.alloc(sizeof(uint64_t) * nnz));
        F3S_CUDA_TRY(keys_alt.alloc(sizeof(uint64_t) * nnz));
        F3S_CUDA_TRY(pos.alloc(sizeof(int32_t) * nnz));
        k_make_keys<<<grid_for((int64_t)n_rows * 32, 256), 256, 0, stream>>>(
            row_ptr, col_idx, n_rows, n_cols, colbits, ends[0], keys.as<uint64_t>(), flag.as<int32_t>());
        count_launch();
        F3S_CUDA_TRY(cudaGetLastError());
        size_t tb_sort = 0, tb_scan = 0;
        cub::DoubleBuffer<uint64_t> db(keys.as<uint64_t>(), keys_alt.as<uint64_t>());
        F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, db, (int64_t)nnz, 0, key_bits, stream));
        F3S_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb_scan, pos.as<int32_t>(), pos.as<int32_t>(), (int64_t)nnz, stream));
        F3S_CUDA_TRY(temp.alloc(std::max(tb_sort, tb_scan)));
        size_t tb = tb_sort;
        F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(temp.p, tb, db, (int64_t)nnz, 0, key_bits, stream));
        count_launch(4);
        const uint64_t* sorted = db.Current();
        k_heads<<<grid_for(nnz, 256), 256, 0, stream>>>(sorted, nnz, pos.as<int32_t>());
        count_launch();
        tb = tb_scan;
        F3S_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp.p, tb, pos.as<int32_t>(), pos.as<int32_t>(), (int64_t)nnz, stream));
        count_launch();
        int32_t hW = 0;
        F3S_CUDA_TRY(cudaMemcpyAsync(&hW, pos.as<int32_t>() + nnz - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        F3S_CUDA_TRY(cudaMemcpyAsync(&hflag, flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        F3S_CUDA_TRY(cudaStreamSynchronize(stream));
        if (hflag & 2) { set_error("a column index is outside [0, n_cols)"); return F3S_ERR_INVALID_CSR; }
        W = hW;
        F3S_CUDA_TRY(cudaMalloc(&plan->cols, sizeof(int32_t) * std::max<int64_t>(W, 1)));
        F3S_CUDA_TRY(cudaMalloc(&plan->masks, sizeof(uint16_t) * std::max<int64_t>(W, 1)));
        k_fill<<<grid_for(nnz, 256), 256, 0, stream>>>(sorted, pos.as<int32_t>(), nnz, colbits, plan->cols,
                                                        plan->masks, widths.as<int32_t>(), d_pop);
        count_launch();
        F3S_CUDA_TRY(cudaGetLastError());
    } else {
        F3S_CUDA_TRY(cudaMalloc(&plan->cols, sizeof(int32_t)));
        F3S_CUDA_TRY(cudaMalloc(&plan->masks, sizeof(uint16_t)));
    }
    plan->total_cols = W;

    // ---- 3. rw_ptr = exclusive scan of widths; LPT order -------------------------------------
    F3S_CUDA_TRY(cudaMalloc(&plan->rw_ptr, sizeof(int32_t) * (size_t)(R + 1)));
    F3S_CUDA_TRY(cudaMalloc(&plan->rw_order, sizeof(int32_t) * (size_t)std::max(R, 1)));
    F3S_CUDA_TRY(cudaMalloc(&plan->rw_natural, sizeof(int32_t) * (size_t)std::max(R, 1)));
    {
        size_t tb_scan = 0;
        F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, widths.as<int32_t>(), plan->rw_ptr, R + 1, stream));
        DevBuf t2;
        F3S_CUDA_TRY(t2.alloc(tb_scan));
        F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t2.p, tb_scan, widths.as<int32_t>(), plan->rw_ptr, R + 1, stream));
        count_launch();
    }
    if (R > 0) {
        DevBuf ok, ok_alt, t3;
        F3S_CUDA_TRY(ok.alloc(sizeof(uint64_t) * R));
        F3S_CUDA_TRY(ok_alt.alloc(sizeof(uint64_t) * R));
        k_order_keys<<<grid_for(R, 256), 256, 0, stream>>>(plan->rw_ptr, R, ok.as<uint64_t>(), plan->rw_natural);
        count_launch();
        cub::DoubleBuffer<uint64_t> db(ok.as<uint64_t>(), ok_alt.as<uint64_t>());
        size_t tb = 0;
        F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, R, 0, 64, stream));
        F3S_CUDA_TRY(t3.alloc(tb));
        F3S_CUDA_TRY(cub::DeviceRadixSort::SortKeys(t3.p, tb, db, R, 0, 64, stream));
        count_launch(4);
        k_order_extract<<<grid_for(R, 256), 256, 0, stream>>>(db.Current(), R, plan->rw_order);
        count_launch();
        F3S_CUDA_TRY(cudaGetLastError());
    }
    // 8-aligned window starts of the kernel layout
    DevBuf w8, rw8, t4;
    F3S_CUDA_TRY(w8.alloc(sizeof(int32_t) * (size_t)(R + 1)));
    F3S_CUDA_TRY(rw8.alloc(sizeof(int32_t) * (size_t)(R + 1)));
    k_width8<<<grid_for(R + 1, 256), 256, 0, stream>>>(plan->rw_ptr, R, w8.as<int32_t>());
    count_launch();
    {
        size_t tb = 0;
        F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, w8.as<int32_t>(), rw8.as<int32_t>(), R + 1, stream));
        F3S_CUDA_TRY(t4.alloc(tb));
        F3S_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t4.p, tb, w8.as<int32_t>(), rw8.as<int32_t>(), R + 1, stream));
        count_launch();
    }

    // ---- 4. statistics (sync #3) --------------------------------------------------------------
    std::vector<int32_t> h_rw(R + 1);
    unsigned long long h_pop = 0;
    int32_t h_w8 = 0;
    F3S_CUDA_TRY(cudaMemcpyAsync(&h_w8, rw8.as<int32_t>() + R, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    F3S_CUDA_TRY(cudaMemcpyAsync(h_rw.data(), plan->rw_ptr, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToHost, stream));
    F3S_CUDA_TRY(cudaMemcpyAsync(&h_pop, d_pop, sizeof(h_pop), cudaMemcpyDeviceToHost, stream));
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    int64_t tcb = 0;
    int32_t maxw = 0;
    for (int32_t k = 0; k < R; ++k) {
        int32_t w = h_rw[k + 1] - h_rw[k];
        tcb += (w + 7) / 8;
        maxw = std::max(maxw, w);
    }
    plan->total_tcb8 = tcb;
    plan->max_width = maxw;
    plan->nnz = (int64_t)h_pop;  // deduplicated nnz = total mask popcount
    plan->total_cols8 = h_w8;
    F3S_CUDA_TRY(cudaMalloc(&plan->kcols, sizeof(int32_t) * std::max<int64_t>(h_w8, 8)));
    F3S_CUDA_TRY(cudaMalloc(&plan->kmasks, sizeof(uint16_t) * std::max<int64_t>(h_w8, 8)));
    F3S_CUDA_TRY(cudaMalloc(&plan->meta_lpt, sizeof(int4) * std::max(R, 1)));
    F3S_CUDA_TRY(cudaMalloc(&plan->meta_nat, sizeof(int4) * std::max(R, 1)));
    if (R > 0) {
        k_kernel_layout<<<grid_for((int64_t)R * 32, 256), 256, 0, stream>>>(
            plan->rw_ptr, rw8.as<int32_t>(), plan->cols, plan->masks, plan->rw_order, R, plan->kcols, plan->kmasks,
            plan->meta_lpt, plan->meta_nat);
        count_launch();
        F3S_CUDA_TRY(cudaGetLastError());
    }
    // heavy-window split list (host: the widths are already here; the order is R ints)
    plan->h_rw = std::move(h_rw);
    plan->h_rw8.resize(R + 1);
    plan->h_order.resize(R);
    if (R > 0) {
        F3S_CUDA_TRY(cudaMemcpyAsync(plan->h_rw8.data(), rw8.as<int32_t>(), sizeof(int32_t) * (R + 1),
                                     cudaMemcpyDeviceToHost, stream));
        F3S_CUDA_TRY(cudaMemcpyAsync(plan->h_order.data(), plan->rw_order, sizeof(int32_t) * R,
                                     cudaMemcpyDeviceToHost, stream));
    }
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    {
        // default: a window is split when it alone exceeds half of an SM's even share of all
        // chunks (counted for one head; more heads only make the share larger).  A row-shard
        // plan counts only its own chunks; multi-GPU callers reset the bound from the global
        // count (f3s_default_split_chunks + f3s_plan_set_split) so shards split like the 1-GPU plan.
        int64_t chunks = 0;
        for (int32_t k = 0; k < R; ++k)
            chunks += std::max<int64_t>(1, (plan->h_rw[k + 1] - plan->h_rw[k] + kSplitChunkCols - 1) / kSplitChunkCols);
        plan->total_chunks = chunks;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plan->device);
        f3s_status st = build_split(plan, default_split_chunks(chunks, sms));
        if (st != F3S_OK) return st;
    }
    F3S_CUDA_TRY(cudaEventRecord(ev1, stream));
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));  // the plan is complete when f3s_plan returns
    F3S_CUDA_TRY(cudaEventElapsedTime(&plan->build_ms, ev0, ev1));
    plan->device_bytes = (int64_t)sizeof(int32_t) * (2 * R + 1 + R) + (int64_t)sizeof(int4) * 2 * R +
                         (int64_t)(sizeof(int32_t) + sizeof(uint16_t)) * (std::max<int64_t>(W, 1) + h_w8);
    guard.ok = true;
    *out = plan;
    return F3S_OK;
}

f3s_status build_split(Plan* p, int32_t chunks) {
    const int32_t R = p->num_rw;
    std::vector<int4> meta, info;
    meta.reserve(R);
    int32_t groups = 0, pieces = 0;
    int32_t heavy_prefix = 0;  // entries up to the last one of >= kHeavyChunks chunks
    int32_t heavy_lpt = 0;     // the same over the unsplit list
    auto note = [&](int64_t nch) {
        if (nch >= kHeavyChunks) heavy_prefix = (int32_t)meta.size();
    };
    for (int32_t i = 0; i < R; ++i) {
        const int32_t k = p->h_order[i], w = p->h_rw[k + 1] - p->h_rw[k], b8 = p->h_rw8[k];
        const int64_t nch = std::max<int64_t>(1, (w + kSplitChunkCols - 1) / kSplitChunkCols);
        if (nch >= kHeavyChunks) heavy_lpt = i + 1;
        if (chunks <= 0 || nch <= chunks) {
            meta.push_back(make_int4(k, b8, w, 0));
            note(nch);
            continue;
        }
        const int32_t np = (int32_t)((nch + chunks - 1) / chunks), step = chunks * kSplitChunkCols;
        if ((int64_t)pieces + np >= (1 << 23)) { set_error("split: too many pieces"); return F3S_ERR_UNSUPPORTED; }
        info.push_back(make_int4(pieces, np, k, 0));
        for (int32_t j = 0; j < np; ++j) {
            const int32_t c0 = j * step;
            meta.push_back(make_int4(k, b8 + c0, std::min(step, w - c0), ++pieces));
            note((std::min(step, w - c0) + kSplitChunkCols - 1) / kSplitChunkCols);
        }
        ++groups;
    }
    // build the new lists completely before swapping them in: on failure the plan keeps its
    // previous (consistent) split
    DevBuf nmeta, ninfo;
    F3S_CUDA_TRY(nmeta.alloc(sizeof(int4) * std::max<size_t>(meta.size(), 1)));
    F3S_CUDA_TRY(ninfo.alloc(sizeof(int4) * std::max<size_t>(info.size(), 1)));
    if (!meta.empty())
        F3S_CUDA_TRY(cudaMemcpy(nmeta.p, meta.data(), sizeof(int4) * meta.size(), cudaMemcpyHostToDevice));
    if (!info.empty())
        F3S_CUDA_TRY(cudaMemcpy(ninfo.p, info.data(), sizeof(int4) * info.size(), cudaMemcpyHostToDevice));
    cudaFree(p->meta_sub);
    cudaFree(p->ginfo);
    p->meta_sub = nmeta.as<int4>();
    p->ginfo = ninfo.as<int4>();
    nmeta.p = ninfo.p = nullptr;
    p->split_chunks = chunks;
    p->n_sub = (int32_t)meta.size();
    p->n_groups = groups;
    p->n_pieces = pieces;
    p->n_heavy_sub = heavy_prefix;
    // entries up to the last wide window or split piece (a split window's last piece can be narrow):
    // everything after it is an unsplit window of <= 32 columns
    int32_t wide = 0;
    for (int32_t i = 0; i < (int32_t)meta.size(); ++i)
        if (meta[i].z > 32 || meta[i].w != 0) wide = i + 1;
    p->n_wide_sub = wide;
    p->n_heavy_lpt = heavy_lpt;
    return F3S_OK;
}

}  // namespace f3s
