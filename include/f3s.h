/*
 * f3s.h — C ABI of the B200-native fused 3S sparse-attention library (libf3s.so).
 *
 *   O = softmax_row( scale * (Q K^T) ⊙ A ) V      per head,
 *
 * Eq.1 of Fused3S decomposed as SDDMM -> row softmax -> SpMM
 * (PAPER.md:116-120), computed in one fused kernel (Alg.1).
 *
 * Conventions (readings of the paper, listed in DESIGN.md §Readings):
 *  - A is binary: only its support matters; duplicate (row, col) entries are merged and
 *    rows may be unsorted.  The softmax runs over the support of row i
 *    only: non-edges get weight exactly 0.  No self-loops are added.
 *  - Rows of A with no entries produce O rows of exact zeros (Alg.1 line 24, divides
 *    by l_o = 0; reading c4).
 *  - Precision follows Tab.mixedp: Q, K, V in fp16 (or bf16); scores,
 *    softmax statistics and O accumulation in fp32; normalised scores cast to the input
 *    dtype before the second contraction; O written in fp32.
 *  - Every call returns f3s_status; nothing throws across this boundary.  Detail for the
 *    last failure on the calling thread is in f3s_last_error().
 *
 * Memory: "device" pointers are CUDA device pointers on the current device; "host"
 * pointers are ordinary host memory (pinned host memory makes the _host call faster).
 * The library never retains caller pointers past the call, except that kernels launched by
 * f3s_attention read Q/K/V and write O asynchronously on `stream`.
 */
#ifndef F3S_H_
#define F3S_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* identical to the CUDA runtime's own declaration (driver_types.h) */
typedef struct CUstream_st* cudaStream_t;

typedef struct f3s_plan_impl* f3s_plan_t; /* opaque; owns device memory until f3s_plan_destroy */

typedef enum {
    F3S_OK = 0,
    F3S_ERR_INVALID_VALUE = 1, /* bad pointer / negative size / heads < 1 / non-finite scale   */
    F3S_ERR_INVALID_CSR = 2,   /* row_ptr not monotone (or row_ptr[0] != 0 for f3s_plan), or a
                                  column index outside [0, n_cols)                             */
    F3S_ERR_UNSUPPORTED = 3,   /* d not in {64, 128}, sizes >= 2^31, misaligned tensors        */
    F3S_ERR_OUT_OF_MEMORY = 4,
    F3S_ERR_CUDA = 5,          /* a CUDA runtime/driver call failed; see f3s_last_error()     */
    F3S_ERR_INTERNAL = 6
} f3s_status;

/* Element type of Q, K, V.  F3S_E4M3 (OCP FP8 E4M3, torch.float8_e4m3fn; SURVEY 8(f) f4 "FP8 K/V
 * gathers", FP8 being the paper's future work): d in {64, 128}, f3s_attention /
 * f3s_attention_host(_async) / the DEFAULT and NO_REORDER variants only.  S is exact on the
 * given fp8 values (fp32 accumulate); P is rounded to e4m3 for the SpMM (l.19), so |O - O_exact|
 * <= 2^-4 * max |V_j| over the row's neighbours (plus fp32 rounding), reading c24. */
typedef enum { F3S_FP16 = 0, F3S_BF16 = 1, F3S_E4M3 = 2 } f3s_dtype;

typedef struct {
    int32_t n_rows;       /* rows of A (local rows for f3s_plan_rows)                          */
    int32_t n_cols;       /* columns of A                                                      */
    int32_t num_rw;       /* R = ceil(n_rows / 16) row windows (r = 16)          */
    int32_t max_width;    /* largest compacted width of a row window                           */
    int64_t nnz;          /* deduplicated nonzeros of A = sum of mask popcounts                */
    int64_t total_cols;   /* W = sum of compacted widths                        */
    int64_t total_tcb8;   /* sum over RWs of ceil(w/8): 16x8 TCB count  */
    int64_t device_bytes; /* device memory owned by the plan                                   */
    float build_ms;       /* device time of the plan build                                     */
    float reserved;
    int32_t split_chunks; /* heavy-window split: pieces of at most this many 128-column chunks  */
    int32_t split_groups; /* row windows that are split      */
    int64_t total_chunks; /* sum over windows of max(1, ceil(w / 128)): kernel chunks of one head  */
} f3s_plan_info;

/*
 * Build the row-window plan of an n x n binary A given in CSR on the DEVICE (§3.1,
 * PAPER.md:206-216, plus the RW reordering of PAPER.md:402-405):
 *   for RW k (rows 16k .. 16k+15):  cols_k = ascending unique column ids of those rows
 *   (compaction; sptd analogue), masks_k[p] bit i set iff (16k+i, cols_k[p])
 *   is in A (bitmap analogue), rw_ptr = prefix sum of widths (tro analogue),
 *   rw_order = RW indices sorted by ceil(w/8) descending, ties by index ascending.
 *
 *  row_ptr  device int32[n+1], row_ptr[0] == 0, non-decreasing.     (read-only, caller-owned)
 *  col_idx  device int32[row_ptr[n]], each in [0, n).                (read-only, caller-owned)
 *  n        number of nodes, 0 <= n < 2^31.  n == 0 gives a valid empty plan.
 *  stream   work is ordered on this stream; the call synchronises the stream (twice) to size
 *           the plan's buffers and to report CSR errors, so both inputs may be freed on return.
 *  out      receives the plan handle (set to NULL on failure).
 * Errors: INVALID_VALUE, INVALID_CSR (detected on the device), OUT_OF_MEMORY, CUDA.
 */
f3s_status f3s_plan(const int32_t* row_ptr, const int32_t* col_idx, int32_t n, cudaStream_t stream,
                    f3s_plan_t* out);

/*
 * Plan for a row block of a rectangular A (n_rows x n_cols): the multi-GPU shard form.
 * Row r of the block has entries col_idx[row_ptr[r] .. row_ptr[r+1]) with row_ptr[0] >= 0
 * allowed to be non-zero, so a caller can pass `global_row_ptr + row_begin` and the global
 * col_idx without copying.  Column ids are global (in [0, n_cols)).  If row_begin is a
 * multiple of 16, every row window equals the corresponding window of the global plan, so
 * per-row results are bitwise identical to the single-GPU call.
 * Other semantics as f3s_plan.
 */
f3s_status f3s_plan_rows(const int32_t* row_ptr, const int32_t* col_idx, int32_t n_rows, int32_t n_cols,
                         cudaStream_t stream, f3s_plan_t* out);

/* Free the plan's device memory.  No call using the plan may still be in flight.  NULL is OK. */
f3s_status f3s_plan_destroy(f3s_plan_t plan);

/* Sizes and statistics of a plan (host struct written by the call). */
f3s_status f3s_plan_get_info(f3s_plan_t plan, f3s_plan_info* info);

/*
 * Copy the canonical plan arrays to HOST memory (synchronous): rw_ptr[R+1], cols[W],
 * masks[W] (uint16, bit i = row 16k+i), rw_order[R].  Any pointer may be NULL to skip it.
 * These arrays are independent of the kernel's tile size and are what the tests compare
 * bit-exactly with the oracle's block builder.
 */
/*
 * Heavy row-window split (load balance under degree skew; the paper's "assigning multiple
 * thread blocks per row window").  f3s_attention (default variant) processes
 * a row window of more than max_chunks 128-column chunks as pieces of max_chunks chunks on
 * different CTAs; each piece leaves its partial (row max, row sum, unnormalised O) in a
 * per-call stream-ordered scratch buffer and a second launch merges the pieces of every split
 * window in piece order (O = sum_p 2^{m_p - M} O_p / sum_p 2^{m_p - M} l_p), so results stay
 * bitwise deterministic.  f3s_plan picks f3s_default_split_chunks(info.total_chunks, SMs); this
 * call rebuilds the piece list with another bound (max_chunks <= 0: never split).  A row-shard
 * plan (f3s_plan_rows) counts only its own chunks: to split exactly like the single-GPU plan
 * (and so keep shard results bitwise equal to it) pass the bound of the GLOBAL chunk count,
 * f3s_default_split_chunks(sum of every shard's total_chunks, SMs).  Host-synchronous; not to be
 * called while attention calls on the plan are in flight.  On failure the plan keeps its
 * previous piece list.
 * Errors: INVALID_VALUE (NULL plan), UNSUPPORTED (more than 2^23 pieces in total), OUT_OF_MEMORY, CUDA.
 */
f3s_status f3s_plan_set_split(f3s_plan_t plan, int32_t max_chunks);

/* The default split bound: max(16, ceil(total_chunks / (2 * 8 * num_sms))): a window is split when
 * it alone exceeds half of an SM's even share of all chunks spread over 8 GPUs (the largest row-
 * shard count the library targets), so single-GPU and shard plans of up to 8 GPUs split alike.
 * Pure host arithmetic. */
int32_t f3s_default_split_chunks(int64_t total_chunks, int32_t num_sms);

f3s_status f3s_plan_export(f3s_plan_t plan, int32_t* rw_ptr, int32_t* cols, uint16_t* masks, int32_t* rw_order);

/*
 * The fused 3S pass (Alg.1) on sm_100a: per row window and head, gathers
 * of K and V rows by the compacted column list (Alg.1 l.7-8) into 128B-swizzled shared-memory
 * tiles (16-byte cp.async; the Q tile and the O tile move by TMA),
 * S^T = K_c Q_w^T on tcgen05 tensor cores into TMEM (l.13), bitmap mask (l.14), online
 * softmax in fp32 (l.16-18), P cast to the input dtype (l.19), O^T += V_c^T P^T on tcgen05
 * (l.21-22), O = O / l written once (l.24).  Row windows are scheduled longest-first
 * from a persistent work queue.
 *
 *  Q      device [n_rows, heads, d] dtype, contiguous, 16-byte aligned
 *  K, V   device [n_cols, heads, d] dtype, contiguous, 16-byte aligned
 *  O      device [n_rows, heads, d] float32, contiguous; must not alias Q/K/V
 *  scale  multiplies Q K^T before the softmax (scale = 1 reproduces Eq.1; 1/sqrt(d) for GT)
 *  heads  >= 1;  d in {64, 128};  dtype F3S_FP16, F3S_BF16 or F3S_E4M3
 * The library cannot see allocation sizes: Q/O must hold n_rows*heads*d elements and K/V
 * n_cols*heads*d (the Python binding checks shapes and dtypes before calling).
 * Runs on the plan's device (the calling thread's current device is restored on return).
 * Asynchronous on `stream`; only launch-time errors are reported (device faults surface at
 * the caller's next synchronisation, CUDA convention).  Each call owns its work-queue counter
 * (a stream-ordered allocation), so calls may be in flight on any number of streams and CUDA
 * graphs.  Bitwise deterministic.
 */
f3s_status f3s_attention(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                         int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);

/*
 * f3s_attention with K and V rows at an arbitrary row stride (the multi-GPU form: one all-gather
 * of an interleaved [n_cols, 2, heads, d] buffer replicates K and V together, so K = buf,
 * V = buf + heads*d, kv_row_stride = 2*heads*d).  Row j of K is K + j*kv_row_stride elements
 * (likewise V); kv_row_stride >= heads*d and a multiple of 16 bytes.  Default variant; otherwise
 * as f3s_attention.  Errors: as f3s_attention; INVALID_VALUE / UNSUPPORTED for a bad stride.
 */
f3s_status f3s_attention_kv(f3s_plan_t plan, const void* Q, const void* K, const void* V, int64_t kv_row_stride,
                            float* O, float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);

/*
 * f3s_attention on row-strided inputs: row i of Q is Q + i*q_row_stride elements, row j of K (V)
 * is K + j*kv_row_stride (V + j*kv_row_stride); each stride >= heads*d and a multiple of 16 bytes
 * (0 = heads*d).  Lets the fused pass read Q, K, V straight out of one projection GEMM output
 * [n, 3, heads, d] (Q = buf, K = buf + heads*d, V = buf + 2*heads*d, both strides 3*heads*d) --
 * the Graph Transformer layer of PAPER.md:683-694.  Default variant; otherwise as f3s_attention.
 */
f3s_status f3s_attention_strided(f3s_plan_t plan, const void* Q, int64_t q_row_stride, const void* K, const void* V,
                                 int64_t kv_row_stride, float* O, float scale, int32_t heads, int32_t d,
                                 f3s_dtype dtype, cudaStream_t stream);

/*
 * Column-block form for overlapping the multi-GPU K/V exchange with compute (
 * rows are independent, and the online softmax of Alg.1 l.16-21 is order-independent
 * up to rounding): `plan` covers only the columns of one K/V block (f3s_plan_rows over the CSR
 * entries whose column lies in the block, global column ids), so the block can be processed as
 * soon as its K/V rows have arrived.  Writes, for every row i and head h of the plan,
 *   O_part[i, h, :] = sum_j 2^(s_ij - m_ih) v_j   (unnormalised; s in log2 units incl. scale)
 *   ml_part[i, h]   = (m_ih, l_ih = sum_j 2^(s_ij - m_ih))    (two floats; m = -8.5e37, l = 0 and
 *                     O = 0 for a row with no entry in the block)
 * f3s_attention_merge then combines the blocks.  K/V rows at kv_row_stride elements (0: heads*d).
 * max_ctas > 0 caps the persistent grid (leaving SMs to a collective running concurrently).
 *  O_part  device float [n_rows, heads, d];  ml_part device float [n_rows, heads, 2] (8-byte aligned)
 * Errors: as f3s_attention; INVALID_VALUE for NULL ml_part, max_ctas < 0 or a bad stride.
 */
f3s_status f3s_attention_partial(f3s_plan_t plan, const void* Q, const void* K, const void* V, int64_t kv_row_stride,
                                 float* O_part, float* ml_part, float scale, int32_t heads, int32_t d, f3s_dtype dtype,
                                 int32_t max_ctas, cudaStream_t stream);

/*
 * O = merge of `parts` column-block partials, in part order (deterministic):
 *   M = max_g m_g,  l = sum_g 2^(m_g - M) l_g,  O = sum_g 2^(m_g - M) O_g / l   (0 if l = 0),
 * i.e. Alg.1's rescaling (l.18, l.21) and final division (l.24) applied once per block.
 *  O_parts  device float [parts][n_rows][heads][d];  ml_parts device float [parts][n_rows][heads][2]
 *  O        device float [n_rows][heads][d];  1 <= parts <= 32;  d in {64, 128}.
 */
f3s_status f3s_attention_merge(int32_t parts, const float* O_parts, const float* ml_parts, int64_t n_rows,
                               int32_t heads, int32_t d, float* O, cudaStream_t stream);

/*
 * Backward of f3s_attention ("SpMM and SDDMM operations in reverse order",
 * PAPER.md:752): for O = softmax_row(scale * (Q K^T) (.) A) V and dO = dL/dO,
 *   dp_ij = dO_i . v_j,  D_i = sum_j p_ij dp_ij,  ds_ij = p_ij (dp_ij - D_i),
 *   dQ_i = scale sum_j ds_ij k_j,  dK_j = scale sum_i ds_ij q_i,  dV_j = sum_i p_ij dO_i,
 * with p the exact fp32 softmax of Eq.1 (the forward's rounding of P to the input dtype is not
 * differentiated).  Tensor-core path (default): the forward in partial mode gives each row's LSE and
 * D = dO . O; a row pass (S^T = K_c Q_w^T, dP^T = V_c dO_w^T, dS^T, dQ^T += K_c^T dS^T on tcgen05,
 * accumulated in TMEM) and a column pass over the plan of A^T (S = Q_c K_w^T, dP = dO_c V_w^T,
 * dV^T += dO_c^T P, dK^T += Q_c^T dS); dO and dS enter the tensor cores rounded to the input dtype.
 * The plan builds its transposed index and the plan of A^T on its first backward call.  Both passes
 * are deterministic (fixed order, no atomics on the data).
 *
 *  Q, K, V   as for f3s_attention (device, [N, H, d] fp16/bf16, 16-byte aligned).
 *  dO        device fp32 [n_rows, H, d];  dQ device fp32 [n_rows, H, d] (written);
 *  dK, dV    device fp32 [n_cols, H, d] (written; for a row-shard plan (f3s_plan_rows) these are
 *            the shard's partial sums, to be all-reduced by the caller).
 * Asynchronous on `stream` (stream-ordered scratch of about n_rows * H * (6 d + 16) bytes).
 * Errors: as f3s_attention; INVALID_VALUE for NULL dO/dK/dV.
 */
f3s_status f3s_attention_backward(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* dO,
                                  float* dQ, float* dK, float* dV, float scale, int32_t heads, int32_t d,
                                  f3s_dtype dtype, cudaStream_t stream);
/*
 * Training forward: O exactly as f3s_attention (bitwise: the same kernel and
 * rounding) plus each row's softmax statistics, which f3s_attention_backward_saved consumes instead
 * of recomputing the forward.  ml[i][h] = (m, l): m the row maximum of scale * log2(e) * q_i . k_j
 * over the row's entries (Alg.1 l.16, in log2 units; -8.5e37 for an empty row), l = sum_j
 * 2^(s_ij - m) (l.17; 0 for an empty row), so LSE_i = m + log2(l) in the same units.
 *  O   device float [n_rows, heads, d];  ml device float [n_rows, heads, 2] (8-byte aligned).
 * Errors: as f3s_attention; INVALID_VALUE for NULL ml.
 */
f3s_status f3s_attention_fwd(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float* ml,
                             float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);

/*
 * f3s_attention_backward with the forward's saved outputs (O, ml from f3s_attention_fwd on the same
 * plan, Q, K, V, scale): the same two tensor-core passes without the forward recomputation (the
 * backward of a training step: PAPER.md:752).  D_i = dO_i . O_i and LSE_i = m_i + log2(l_i).
 *  O   device float [n_rows, heads, d] (16-byte aligned);  ml device float [n_rows, heads, 2].
 *  Other arguments as f3s_attention_backward (stream-ordered scratch of about n_rows * H * (2 d + 8)
 *  bytes).  Errors: as f3s_attention_backward; INVALID_VALUE for NULL O/ml.
 */
f3s_status f3s_attention_backward_saved(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* O,
                                        const float* ml, const float* dO, float* dQ, float* dK, float* dV, float scale,
                                        int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);

/*
 * f3s_attention_backward_saved in the input dtype (F3S_FP16 / F3S_BF16): dO is given in it (device
 * [n_rows, heads, d], 16-byte aligned; the tensor cores read it in place and D_i = dO_i . O_i uses its
 * values) and dQ [n_rows, heads, d], dK, dV [n_cols, heads, d] are written in it (the fp32 TMEM
 * accumulators rounded once, RNE) -- a 16-bit layer's gradients with no conversions and half the
 * gradient bytes.  Errors: as f3s_attention_backward_saved.
 */
f3s_status f3s_attention_backward_saved_lp(f3s_plan_t plan, const void* Q, const void* K, const void* V,
                                           const float* O, const float* ml, const void* dO, void* dQ, void* dK,
                                           void* dV, float scale, int32_t heads, int32_t d, f3s_dtype dtype,
                                           cudaStream_t stream);

/* variant 0: the tensor-core path of f3s_attention_backward; 1: the CUDA-core two-pass kernels
 * (one warp per row / column walking its entries in fp32: online max/sum/D, then p, ds; the
 * reference for the tensor-core path).  Errors: as f3s_attention_backward; INVALID_VALUE for
 * another variant. */
f3s_status f3s_attention_backward_ex(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* dO,
                                     float* dQ, float* dK, float* dV, float scale, int32_t heads, int32_t d,
                                     f3s_dtype dtype, int32_t variant, cudaStream_t stream);

/* Kernel variants for ablations (bench.py --variant); f3s_attention uses F3S_VARIANT_DEFAULT. */
typedef enum {
    F3S_VARIANT_DEFAULT = 0, /* tcgen05 kernel, LPT-ordered persistent queue, heavy-window split */
    F3S_VARIANT_NO_REORDER = 1, /* same kernel, row windows in natural order */
    F3S_VARIANT_SIMT = 2,    /* CUDA-core reference kernel of the same dataflow (no tensor core) */
    F3S_VARIANT_ONE_HEAD = 3 /* tcgen05 kernel with one head per chunk even where the default packs
                                4 heads of windows <= 32 columns wide into one chunk (d = 64)   */
} f3s_variant;

f3s_status f3s_attention_ex(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                            int32_t heads, int32_t d, f3s_dtype dtype, f3s_variant variant, cudaStream_t stream);

/*
 * Diagnostics (F3S_TRACE): the default kernel with a device buffer trace[grid][trace_chunks][8]
 * of uint64 globaltimer stamps per CTA and chunk: 0 ids/masks requested, 1 gathers issued,
 * 2 MMA1 issued, 3 scores seen, 4 P written, 5 MMA2 issued, 6 O seen, 7 rows stored (last
 * chunk of an item).  grid > 0 overrides the persistent grid size (0 = default).
 */
f3s_status f3s_attention_trace(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                               int32_t heads, int32_t d, f3s_dtype dtype, f3s_variant variant, uint64_t* trace,
                               int32_t trace_chunks, int32_t grid, cudaStream_t stream);

/*
 * End-to-end form with HOST buffers: copies Q, K, V host->device, runs f3s_attention, copies
 * O device->host and synchronises `stream`.  Device staging buffers are owned by the plan and
 * reused across calls.  Q: host [n_rows,heads,d], K/V: host [n_cols,heads,d], O: host float32.
 */
f3s_status f3s_attention_host(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O,
                              float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);
/* The same, stream-ordered: returns once the copies, the fused call and the read-back are
 * enqueued; O is valid after `stream` completes.  The device staging buffer belongs to the
 * stream (one per stream and plan), so calls on two streams overlap one call's host-to-device
 * copies with the other's device-to-host copy (full-duplex PCIe/NVLink-C2C).  With pageable host
 * memory the copies are synchronous (CUDA semantics); use pinned buffers to overlap. */
f3s_status f3s_attention_host_async(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O,
                                    float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream);

/*
 * Host partitioner for multi-GPU runs: split rows [0, n) into `parts` contiguous ranges whose
 * boundaries are multiples of 16 (row-window aligned, except bounds[parts] = n), balancing
 * nnz: bounds[p] is the window boundary whose prefix nnz is closest to p * nnz / parts.
 *  row_ptr_host  host int32[n+1] (row_ptr[0] may be non-zero)
 *  bounds        host int32[parts+1] written: 0 = bounds[0] <= ... <= bounds[parts] = n
 */
f3s_status f3s_partition_rows(const int32_t* row_ptr_host, int32_t n, int32_t parts, int32_t* bounds);

/* Same, but only cutting at the given candidate boundaries (e.g. graph starts in batched
 * mode): cuts[n_cuts] ascending in [0, n]. */
f3s_status f3s_partition_at(const int32_t* row_ptr_host, int32_t n, const int32_t* cuts, int32_t n_cuts,
                            int32_t parts, int32_t* bounds);

const char* f3s_status_string(f3s_status s);
const char* f3s_last_error(void); /* thread-local detail of the last failure, "" if none */

/* Number of kernels the library launched since load (bench.py's gpu_launches evidence). */
int64_t f3s_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* F3S_H_ */
