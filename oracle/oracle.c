/*
 * oracle.c — CPU oracle for the fused 3S hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2505_08098_b200/) never does.
 * It shares no code, headers or helpers with the CUDA path.
 *
 * Two functions, each the plain definition of what the path computes:
 *
 *  oracle_attention  O = softmax_row((Q K^T) ⊙ A) V  per head, Eq.1,
 *                    decomposed as SDDMM / softmax / SpMM with the
 *                    max-stabilised softmax of Eq.7, in fp64.
 *                    Readings: softmax over the support of A only
 *                    (c1), binary A with duplicates merged (c2), scores scaled by `scale`
 *                    (c3), empty rows give O = 0 (c4), inputs are the exact fp16/bf16
 *                    values (c6).  std exp in fp64 (c8).
 *
 *  oracle_plan       the row-window plan of §3.1: for RW k (rows
 *                    16k..16k+15) the ascending unique columns (compaction), a 16-bit
 *                    row mask per column (bitmap; bit i = row 16k+i, reading c12),
 *                    rw_ptr = prefix of widths (tro analogue) and the RW order
 *                    sorted by TCB count ceil(w/8) descending, ties by index (P:402,
 *                    reading c13).
 *
 *  oracle_attention_backward   dQ, dK, dV of Eq.1 for a given dO,
 *                    the softmax Jacobian and the transposed SDDMM/SpMM written out, in fp64;
 *                    oracle_attention_f64 is the same forward on fp64 inputs (its FD target).
 *
 * Pins: tests/test_oracle.py (dense brute force, torch SDPA in fp64, closed forms,
 * invariants, SPEC worked examples), tests/test_oracle_backward.py (central finite
 * differences, torch autograd of dense masked SDPA in fp64, closed forms).  No function here
 * is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* exact decoding of the stored inputs (Tab.mixedp: Q,K,V are fp16) */
static double oracle_f16(uint16_t h) {
    int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp((double)(m + 1024), e - 25);
    return s ? -v : v;
}
static double oracle_bf16(uint16_t b) {
    uint32_t x = (uint32_t)b << 16;
    float f;
    memcpy(&f, &x, 4);
    return (double)f;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * O[r, h, :] for each selected row r (rows == NULL: all n_rows rows, else the n_sel listed
 * rows, output packed in list order).  Q is [n_rows, H, d], K and V are [n_cols, H, d]
 * (uint16 bit patterns of `dtype`: 0 fp16, 1 bf16).  Returns 0, or 2 on an invalid CSR.
 */
int oracle_attention(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                     int32_t H, int32_t d, int32_t dtype, const uint16_t* Q, const uint16_t* K,
                     const uint16_t* V, double scale, const int32_t* rows, int32_t n_sel, double* O,
                     int32_t n_threads) {
    if (n_rows < 0 || n_cols < 0 || H < 1 || d < 1) return 1;
    int32_t count = rows ? n_sel : n_rows;
    for (int32_t r = 0; r < n_rows; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) return 2;
    int bad = 0;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel reduction(| : bad)
    {
        int32_t cap = 0;
        int32_t* nb = NULL;   /* N_i: sorted unique neighbours of row i */
        double* s = NULL;     /* scores s_j of one head */
        double* qd = (double*)malloc((size_t)d * sizeof(double));
        double* acc = (double*)malloc((size_t)d * sizeof(double));
#pragma omp for schedule(dynamic, 64)
        for (int32_t t = 0; t < count; ++t) {
            int32_t i = rows ? rows[t] : t;
            double* out = O + (size_t)t * H * d;
            int32_t b = row_ptr[i], e = row_ptr[i + 1], deg = e - b;
            if (deg > cap) {
                cap = deg;
                nb = (int32_t*)realloc(nb, (size_t)cap * sizeof(int32_t));
                s = (double*)realloc(s, (size_t)cap * sizeof(double));
            }
            /* binary A: the support of row i, duplicates merged (reading c2) */
            for (int32_t p = 0; p < deg; ++p) {
                nb[p] = col_idx[b + p];
                if (nb[p] < 0 || nb[p] >= n_cols) bad = 1;
            }
            if (bad) continue;
            qsort(nb, (size_t)deg, sizeof(int32_t), cmp_i32);
            int32_t u = 0;
            for (int32_t p = 0; p < deg; ++p)
                if (u == 0 || nb[p] != nb[u - 1]) nb[u++] = nb[p];
            if (u == 0) { /* empty row: O = 0 (reading c4) */
                memset(out, 0, (size_t)H * d * sizeof(double));
                continue;
            }
            for (int32_t h = 0; h < H; ++h) {
                const uint16_t* qi = Q + ((size_t)i * H + h) * d;
                for (int32_t k = 0; k < d; ++k) qd[k] = dtype ? oracle_bf16(qi[k]) : oracle_f16(qi[k]);
                /* SDDMM: s_j = scale * q_i . k_j for j in N_i */
                double m = -INFINITY;
                for (int32_t p = 0; p < u; ++p) {
                    const uint16_t* kj = K + ((size_t)nb[p] * H + h) * d;
                    double dot = 0.0;
                    for (int32_t k = 0; k < d; ++k) dot += qd[k] * (dtype ? oracle_bf16(kj[k]) : oracle_f16(kj[k]));
                    s[p] = scale * dot;
                    if (s[p] > m) m = s[p];
                }
                /* softmax, Eq.7: w_j = exp(s_j - max s), l = sum w_j */
                double l = 0.0;
                for (int32_t p = 0; p < u; ++p) { s[p] = exp(s[p] - m); l += s[p]; }
                /* SpMM: O_i = sum_j w_j v_j / l */
                for (int32_t k = 0; k < d; ++k) acc[k] = 0.0;
                for (int32_t p = 0; p < u; ++p) {
                    const uint16_t* vj = V + ((size_t)nb[p] * H + h) * d;
                    for (int32_t k = 0; k < d; ++k) acc[k] += s[p] * (dtype ? oracle_bf16(vj[k]) : oracle_f16(vj[k]));
                }
                for (int32_t k = 0; k < d; ++k) out[(size_t)h * d + k] = acc[k] / l;
            }
        }
        free(nb);
        free(s);
        free(qd);
        free(acc);
    }
    return bad ? 2 : 0;
}

/* ------------------------------------------------------------------------- */
/* backward ("SpMM and SDDMM operations in      */
/* reverse order")                                                           */
/* ------------------------------------------------------------------------- */

/*
 * Gradients of O = softmax_row(scale * (Q K^T) (.) A) V (Eq.1, same readings c1-c4 as
 * oracle_attention) with respect to Q, K and V, given dO = dL/dO; all values fp64 ([n, H, d]
 * row-major; Q, dO, dQ have n_rows rows, K, V, dK, dV have n_cols rows).  Per row i and head h,
 * with N_i the sorted unique neighbours (empty rows contribute nothing and get dQ_i = 0):
 *   s_j  = scale * q_i . k_j,   p_j = exp(s_j - max s) / sum_t exp(s_t - max s)     (Eq.7)
 *   dp_j = dO_i . v_j                                            (SDDMM of dO with V)
 *   D_i  = sum_j p_j dp_j                                        (= dO_i . O_i)
 *   ds_j = p_j (dp_j - D_i)                                      (softmax Jacobian)
 *   dQ_i = scale * sum_j ds_j k_j                                (SpMM)
 *   dK_j += scale * ds_j q_i,   dV_j += p_j dO_i                 (transposed SpMMs)
 * Rows are visited in order, so the accumulation into dK / dV is deterministic.
 * Returns 0, or 2 on an invalid CSR.
 */
int oracle_attention_backward(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                              int32_t H, int32_t d, const double* Q, const double* K, const double* V,
                              const double* dO, double scale, double* dQ, double* dK, double* dV) {
    if (n_rows < 0 || n_cols < 0 || H < 1 || d < 1) return 1;
    for (int32_t r = 0; r < n_rows; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) return 2;
    memset(dQ, 0, (size_t)n_rows * H * d * sizeof(double));
    memset(dK, 0, (size_t)n_cols * H * d * sizeof(double));
    memset(dV, 0, (size_t)n_cols * H * d * sizeof(double));
    int32_t cap = 0;
    int32_t* nb = NULL;
    double *p = NULL, *dp = NULL;
    int bad = 0;
    for (int32_t i = 0; i < n_rows && !bad; ++i) {
        int32_t b = row_ptr[i], e = row_ptr[i + 1], deg = e - b;
        if (deg > cap) {
            cap = deg;
            nb = (int32_t*)realloc(nb, (size_t)cap * sizeof(int32_t));
            p = (double*)realloc(p, (size_t)cap * sizeof(double));
            dp = (double*)realloc(dp, (size_t)cap * sizeof(double));
        }
        for (int32_t t = 0; t < deg; ++t) {
            nb[t] = col_idx[b + t];
            if (nb[t] < 0 || nb[t] >= n_cols) bad = 1;
        }
        if (bad) break;
        qsort(nb, (size_t)deg, sizeof(int32_t), cmp_i32);
        int32_t u = 0;
        for (int32_t t = 0; t < deg; ++t)
            if (u == 0 || nb[t] != nb[u - 1]) nb[u++] = nb[t];
        for (int32_t h = 0; h < H; ++h) {
            const double* qi = Q + ((size_t)i * H + h) * d;
            const double* gi = dO + ((size_t)i * H + h) * d;
            double m = -INFINITY, l = 0.0, Di = 0.0;
            for (int32_t t = 0; t < u; ++t) {
                const double* kj = K + ((size_t)nb[t] * H + h) * d;
                const double* vj = V + ((size_t)nb[t] * H + h) * d;
                double dot = 0.0, dv = 0.0;
                for (int32_t k = 0; k < d; ++k) { dot += qi[k] * kj[k]; dv += gi[k] * vj[k]; }
                p[t] = scale * dot;
                dp[t] = dv;
                if (p[t] > m) m = p[t];
            }
            for (int32_t t = 0; t < u; ++t) { p[t] = exp(p[t] - m); l += p[t]; }
            for (int32_t t = 0; t < u; ++t) { p[t] /= l; Di += p[t] * dp[t]; }
            double* dqi = dQ + ((size_t)i * H + h) * d;
            for (int32_t t = 0; t < u; ++t) {
                const double ds = p[t] * (dp[t] - Di);
                const double* kj = K + ((size_t)nb[t] * H + h) * d;
                double* dkj = dK + ((size_t)nb[t] * H + h) * d;
                double* dvj = dV + ((size_t)nb[t] * H + h) * d;
                for (int32_t k = 0; k < d; ++k) {
                    dqi[k] += scale * ds * kj[k];
                    dkj[k] += scale * ds * qi[k];
                    dvj[k] += p[t] * gi[k];
                }
            }
        }
    }
    free(nb);
    free(p);
    free(dp);
    return bad ? 2 : 0;
}

/*
 * The forward of Eq.1 on fp64 inputs (same definition as oracle_attention, which reads the
 * exact fp16/bf16 values): the function whose derivative oracle_attention_backward is; used
 * by the finite-difference pins of the backward.
 */
int oracle_attention_f64(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                         int32_t H, int32_t d, const double* Q, const double* K, const double* V, double scale,
                         double* O) {
    if (n_rows < 0 || n_cols < 0 || H < 1 || d < 1) return 1;
    int32_t cap = 0;
    int32_t* nb = NULL;
    double* w = NULL;
    int bad = 0;
    for (int32_t i = 0; i < n_rows && !bad; ++i) {
        int32_t b = row_ptr[i], e = row_ptr[i + 1], deg = e - b;
        if (deg < 0) { bad = 1; break; }
        if (deg > cap) {
            cap = deg;
            nb = (int32_t*)realloc(nb, (size_t)cap * sizeof(int32_t));
            w = (double*)realloc(w, (size_t)cap * sizeof(double));
        }
        for (int32_t t = 0; t < deg; ++t) {
            nb[t] = col_idx[b + t];
            if (nb[t] < 0 || nb[t] >= n_cols) bad = 1;
        }
        if (bad) break;
        qsort(nb, (size_t)deg, sizeof(int32_t), cmp_i32);
        int32_t u = 0;
        for (int32_t t = 0; t < deg; ++t)
            if (u == 0 || nb[t] != nb[u - 1]) nb[u++] = nb[t];
        for (int32_t h = 0; h < H; ++h) {
            double* out = O + ((size_t)i * H + h) * d;
            for (int32_t k = 0; k < d; ++k) out[k] = 0.0;
            if (u == 0) continue;
            const double* qi = Q + ((size_t)i * H + h) * d;
            double m = -INFINITY, l = 0.0;
            for (int32_t t = 0; t < u; ++t) {
                const double* kj = K + ((size_t)nb[t] * H + h) * d;
                double dot = 0.0;
                for (int32_t k = 0; k < d; ++k) dot += qi[k] * kj[k];
                w[t] = scale * dot;
                if (w[t] > m) m = w[t];
            }
            for (int32_t t = 0; t < u; ++t) { w[t] = exp(w[t] - m); l += w[t]; }
            for (int32_t t = 0; t < u; ++t) {
                const double* vj = V + ((size_t)nb[t] * H + h) * d;
                for (int32_t k = 0; k < d; ++k) out[k] += w[t] * vj[k];
            }
            for (int32_t k = 0; k < d; ++k) out[k] /= l;
        }
    }
    free(nb);
    free(w);
    return bad ? 2 : 0;
}

/* ------------------------------------------------------------------------- */
/* plan                                                                      */
/* ------------------------------------------------------------------------- */

typedef struct { int32_t col; int32_t bit; } entry_t;
static int cmp_entry(const void* a, const void* b) {
    const entry_t* x = (const entry_t*)a;
    const entry_t* y = (const entry_t*)b;
    if (x->col != y->col) return (x->col > y->col) - (x->col < y->col);
    return (x->bit > y->bit) - (x->bit < y->bit);
}
typedef struct { int32_t tcb; int32_t idx; } order_t;
/* RW reordering: decreasing TCB count, ties by ascending index (reading c13) */
static int cmp_order(const void* a, const void* b) {
    const order_t* x = (const order_t*)a;
    const order_t* y = (const order_t*)b;
    if (x->tcb != y->tcb) return x->tcb > y->tcb ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/*
 * Build the canonical plan of an n_rows x n_cols binary A.  Arrays are malloc'ed here and
 * released with oracle_free.  rw_ptr[R+1], cols[W], masks[W], rw_order[R], R = ceil(n_rows/16).
 * Returns 0, or 2 if the CSR is invalid (row_ptr[0] != 0, decreasing row_ptr, col out of range).
 */
int oracle_plan(int32_t n_rows, int32_t n_cols, const int32_t* row_ptr, const int32_t* col_idx,
                int32_t** rw_ptr_out, int32_t** cols_out, uint16_t** masks_out, int32_t** rw_order_out,
                int64_t* W_out) {
    if (n_rows < 0 || n_cols < 0) return 1;
    if (n_rows > 0 && row_ptr[0] != 0) return 2;
    for (int32_t r = 0; r < n_rows; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) return 2;
    int64_t nnz = n_rows > 0 ? row_ptr[n_rows] : 0;
    for (int64_t p = 0; p < nnz; ++p)
        if (col_idx[p] < 0 || col_idx[p] >= n_cols) return 2;
    int32_t R = (n_rows + 15) / 16;
    int32_t* rw_ptr = (int32_t*)calloc((size_t)R + 1, sizeof(int32_t));
    int32_t* cols = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t)); /* W <= nnz */
    uint16_t* masks = (uint16_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(uint16_t));
    order_t* ord = (order_t*)malloc((size_t)(R > 0 ? R : 1) * sizeof(order_t));
    entry_t* ent = (entry_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(entry_t));
    if (!rw_ptr || !cols || !masks || !ord || !ent) return 3;
    int64_t W = 0;
    for (int32_t k = 0; k < R; ++k) {
        /* step 1: the row window = rows 16k .. min(16k+16, n_rows)-1 */
        int32_t r0 = 16 * k, r1 = r0 + 16 < n_rows ? r0 + 16 : n_rows;
        int64_t m = 0;
        for (int32_t r = r0; r < r1; ++r)
            for (int32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
                ent[m].col = col_idx[p];
                ent[m].bit = r - r0;
                m++;
            }
        /* step 2: keep only columns with a nonzero, in ascending order (reading c11) */
        qsort(ent, (size_t)m, sizeof(entry_t), cmp_entry);
        for (int64_t p = 0; p < m; ++p) {
            if (p == 0 || ent[p].col != ent[p - 1].col) {
                cols[W] = ent[p].col;
                masks[W] = 0;
                W++;
            }
            /* bitmap: bit i of the column's mask marks row 16k+i (reading c12) */
            masks[W - 1] |= (uint16_t)(1u << ent[p].bit);
        }
        rw_ptr[k + 1] = (int32_t)W;
        /* TCB count t = ceil(w/8) at 16x8 tiles */
        ord[k].tcb = (rw_ptr[k + 1] - rw_ptr[k] + 7) / 8;
        ord[k].idx = k;
    }
    qsort(ord, (size_t)R, sizeof(order_t), cmp_order);
    int32_t* rw_order = (int32_t*)malloc((size_t)(R > 0 ? R : 1) * sizeof(int32_t));
    for (int32_t k = 0; k < R; ++k) rw_order[k] = ord[k].idx;
    free(ord);
    free(ent);
    *rw_ptr_out = rw_ptr;
    *cols_out = cols;
    *masks_out = masks;
    *rw_order_out = rw_order;
    *W_out = W;
    return 0;
}

void oracle_free(void* p) { free(p); }
