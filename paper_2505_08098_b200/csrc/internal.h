// internal.h — shared declarations of libf3s (not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/f3s.h"

namespace f3s {

constexpr int kRowsPerWindow = 16;  // r = 16 (reading c10)

struct Plan {
    int32_t n_rows = 0, n_cols = 0, num_rw = 0, max_width = 0;
    int64_t nnz = 0, total_cols = 0, total_tcb8 = 0, device_bytes = 0;
    float build_ms = 0.f;
    int device = 0;
    // canonical arrays (device)
    int32_t* rw_ptr = nullptr;    // [R+1]
    int32_t* cols = nullptr;      // [W]
    uint16_t* masks = nullptr;    // [W]
    int32_t* rw_order = nullptr;  // [R]  LPT order
    int32_t* rw_natural = nullptr;  // [R] identity order (ablation)
    // kernel layout (derived from the canonical arrays): every window's columns start at a
    // multiple of 8 entries so a chunk's ids/masks are 16-byte aligned for cp.async.bulk;
    // the padding repeats the window's last column with mask 0.
    int64_t total_cols8 = 0;
    int32_t* kcols = nullptr;     // [W8]
    uint16_t* kmasks = nullptr;   // [W8]
    int4* meta_lpt = nullptr;     // [R] {k, start8, width, 0} in LPT order
    int4* meta_nat = nullptr;     // [R] same, natural order (no-reorder ablation)
    // heavy row-window split: the default kernel walks
    // meta_sub, the LPT list with every window of more than split_chunks 128-column chunks cut
    // into pieces of split_chunks chunks (meta_sub[i].w = 1 + global piece index, 0 for an
    // unsplit window); each piece leaves (m, l, O) partials and k_split_merge combines the
    // pieces of split window g, in piece order (ginfo[g] = {first global piece, pieces, k, 0})
    int32_t split_chunks = 0, n_sub = 0, n_groups = 0, n_pieces = 0;
    // the LPT list's heavy prefix: entries up to the last of >= kHeavyChunks chunks; the kernel's
    // work queue hands these out one item per claim (lighter items in batches of 8), so that a
    // run of the heaviest windows is not claimed by one CTA
    int32_t n_heavy_sub = 0;
    // meta_sub entries up to the last window wider than 32 columns or split piece; the entries
    // after it (unsplit windows of <= 32 columns, the LPT tail) can run 4 heads per chunk (head
    // groups, d = 64)
    int32_t n_wide_sub = 0;
    int64_t total_chunks = 0;     // sum over windows of max(1, ceil(w / 128)): one head's kernel chunks
    int4* meta_sub = nullptr;     // [n_sub]
    int4* ginfo = nullptr;        // [n_groups]
    std::vector<int32_t> h_rw, h_rw8, h_order;  // host copies used to (re)build meta_sub
    // transposed index of A for the backward's column pass (built on the first backward call):
    // col_rows[col_ptr[j] .. col_ptr[j+1]) = rows i with (i, j) in A, ascending
    int32_t* col_ptr = nullptr;   // [n_cols + 1]
    int32_t* col_rows = nullptr;  // [nnz]
    int32_t* col_lists = nullptr; // [n_light + n_heavy]: columns with 1..64 rows, then with more
    int32_t n_light = 0, n_heavy = 0, n_heavy8 = 0;  // heavy list = n_heavy8 8-warp columns, then 32-warp ones
    int32_t* heavy_rows = nullptr;    // rows with more than 256 entries (backward row pass)
    uint8_t* heavy_row_flag = nullptr;  // [n_rows]
    int32_t n_heavy_rows = 0;
    // e2e staging buffers for f3s_attention_host(_async): one device buffer per stream (reused by
    // later calls on the same stream, which the stream order makes safe)
    struct Staging {
        cudaStream_t stream;
        void* ptr;
        size_t bytes;
    };
    std::mutex staging_mu;
    std::vector<Staging> staging;
    std::mutex transpose_mu;  // the backward's transposed index is built once, under this lock
    Plan* tplan = nullptr;    // plan of A^T for the tensor-core backward's column pass (built on first use)
    int32_t n_heavy_lpt = 0;  // heavy prefix of the unsplit LPT list (meta_lpt), as n_heavy_sub
};

// Switch the calling thread to `dev` for the scope of a call and restore its device after.
struct DeviceScope {
    int prev = -1;
    cudaError_t enter(int dev) {
        cudaError_t e = cudaGetDevice(&prev);
        if (e != cudaSuccess) { prev = -1; return e; }
        if (prev == dev) { prev = -1; return cudaSuccess; }
        return cudaSetDevice(dev);
    }
    ~DeviceScope() { if (prev >= 0) cudaSetDevice(prev); }
};

// Default heavy-window split bound (f3s.h, f3s_plan_set_split): a window is cut into pieces
// when it alone exceeds half of an SM's even share of all chunks of the (global) problem spread
// over kSplitGpus GPUs -- the largest box the row shards target, so that the single-GPU plan and
// every shard of an up-to-8-GPU run split the same windows (bitwise-equal shard results) and the
// 8-GPU tail is balanced (tools/f1_ab.py: Reddit-shaped, slowest of 8 shards 0.44 -> 0.33 ms; the
// extra pieces cost < 1 % at one GPU).
constexpr int64_t kSplitGpus = 8;
inline int32_t default_split_chunks(int64_t total_chunks, int32_t num_sms) {
    const int64_t sms = (num_sms > 0 ? num_sms : 148) * kSplitGpus;
    const int64_t t = std::max<int64_t>(16, (total_chunks + 2 * sms - 1) / (2 * sms));
    return (int32_t)std::min<int64_t>(t, 0x7FFFFFFF);
}

// Stream-ordered per-call scratch from the library's own memory pool on the current device
// (freed memory stays reserved in the pool -- no release threshold -- so steady-state calls reuse it instead of mapping new
// pages at every call; a pool of its own leaves the caller's default-pool settings alone).
cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t stream);
cudaError_t scratch_free(void* ptr, cudaStream_t stream);

// error reporting (thread-local detail)
void set_error(const std::string& msg);
f3s_status cuda_fail(cudaError_t e, const char* what);
void count_launch(int64_t n = 1);

f3s_status build_plan(const int32_t* row_ptr, const int32_t* col_idx, int32_t n_rows, int32_t n_cols,
                      bool require_zero_base, cudaStream_t stream, Plan** out);

struct AttnArgs {
    const Plan* plan;
    const void* Q;
    const void* K;
    const void* V;
    float* O;
    float scale;
    int heads, d;
    f3s_dtype dtype;
    bool lpt;
    cudaStream_t stream;
    uint64_t* trace = nullptr;  // F3S_TRACE buffer [grid][trace_chunks][8] (diagnostics)
    int32_t trace_chunks = 0;
    int32_t grid_override = 0;
    int32_t expt = 0;           // sensitivity experiments (diagnostics only)
    bool one_head = false;      // F3S_VARIANT_ONE_HEAD: no head groups
    int64_t kv_ld = 0;          // elements between consecutive K (and V) rows; 0 = heads * d
    int64_t q_ld = 0;           // elements between consecutive Q rows; 0 = heads * d
    float* ml_out = nullptr;    // partial mode: [n_rows, heads] (m, l) pairs; O left unnormalised
    bool ml_norm = false;       // with ml_out: O normalised as in f3s_attention (f3s_attention_fwd)
    int32_t max_ctas = 0;       // > 0: at most this many CTAs (SMs left for a concurrent collective)
    int32_t sub_begin = 0, sub_end = -1;  // LPT order: this launch's range of meta_sub entries (-1: to the end)
};

f3s_status launch_attention_sm100(const AttnArgs& a);
// 2-D tensor maps over a row-major [rows, inner] matrix (ld elements between rows); 16-bit / 8-bit
// inputs get 128-byte boxes with the 128-byte swizzle of the UMMA tiles, fp32 an unswizzled box
f3s_status make_map(CUtensorMap* map, const void* base, CUtensorMapDataType type, int64_t inner, int64_t rows,
                    int64_t ld, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz);
f3s_status make_map(CUtensorMap* map, const void* base, f3s_dtype dtype, int64_t inner, int64_t rows, int64_t ld,
                    uint32_t box_rows);
f3s_status launch_fill_ml(float* ml, int64_t rows_heads, cudaStream_t stream);
f3s_status launch_parts_merge(int32_t parts, const float* O_parts, const float* ml_parts, int64_t rows_heads, int32_t d,
                              float* O, cudaStream_t stream);
// (re)build meta_sub / sinfo with pieces of at most `chunks` 128-column chunks (chunks <= 0: no split)
f3s_status build_split(Plan* p, int32_t chunks);
constexpr int kSplitChunkCols = 128;  // column granularity of the split (the kernel's chunk)
constexpr int kHeavyChunks = 8;       // an item of this many chunks is claimed alone (= the claim batch)
f3s_status launch_attention_simt(const AttnArgs& a);
f3s_status build_transpose_plan(Plan& p, cudaStream_t stream);
// O, ml: the saved outputs of f3s_attention_fwd, or NULL (the forward is recomputed in partial mode);
// dO, dQ, dK, dV: fp32, or in the input dtype when dO_lp (f3s_attention_backward_saved_lp)
f3s_status launch_attention_backward_tc(Plan& p, const void* Q, const void* K, const void* V, const float* O,
                                        const float* ml, const void* dO, bool dO_lp, void* dQ, void* dK, void* dV,
                                        float scale, int heads, int d, f3s_dtype dtype, cudaStream_t stream);
f3s_status launch_attention_backward(Plan& p, const void* Q, const void* K, const void* V, const float* dO, float* dQ,
                                     float* dK, float* dV, float scale, int heads, int d, f3s_dtype dtype,
                                     cudaStream_t stream);

}  // namespace f3s

#define F3S_CUDA_TRY(expr)                                        \
    do {                                                          \
        cudaError_t e_ = (expr);                                  \
        if (e_ != cudaSuccess) return ::f3s::cuda_fail(e_, #expr); \
    } while (0)
