/*
 * f3s_inputs — seeded synthetic inputs shared by the CUDA path and the oracle.
 *
 * This module holds NO arithmetic of the method (no scores, softmax, blocking or
 * aggregation).  It only produces:
 *   - graphs in CSR form (int32 row_ptr / col_idx, rows sorted, duplicates removed),
 *     shaped like the paper's datasets (Tab.datasets);
 *   - Q/K/V value tensors from a counter-based splitmix64 stream, rounded RNE to
 *     fp16 or bf16 (precision of Tab.mixedp).
 *
 * Every generator is a pure function of its arguments and seed; results are
 * identical on any host and thread count.  See DESIGN.md "Input recipe".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL

/* splitmix64 finaliser; mix64(seed + (i+1)*GOLDEN) is the i-th output of a
 * sequential splitmix64 stream started at `seed` (SPEC.md:528 idea). */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t rng_at(uint64_t seed, uint64_t i) { return mix64(seed + (i + 1) * GOLDEN); }
/* uniform double in [0,1) with 53 random bits */
static inline double u01(uint64_t z) { return (double)(z >> 11) * (1.0 / 9007199254740992.0); }

/* ------------------------------------------------------------------------- */
/* values                                                                    */
/* ------------------------------------------------------------------------- */

static uint16_t f32_to_f16_rne(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    uint32_t sign = (x >> 16) & 0x8000u;
    uint32_t a = x & 0x7FFFFFFFu;
    if (a >= 0x7F800000u) return (uint16_t)(sign | (a > 0x7F800000u ? 0x7E00u : 0x7C00u));
    if (a >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u); /* >= 65520 rounds to inf */
    if (a < 0x38800000u) {                                     /* below 2^-14: subnormal half */
        float af;
        memcpy(&af, &a, 4);
        float r = af * 16777216.0f; /* exact: scale by 2^24 */
        uint32_t m = (uint32_t)nearbyintf(r); /* RNE (default rounding mode) */
        return (uint16_t)(sign | m);
    }
    uint32_t h = (((a >> 23) - 112u) << 10) | ((a & 0x7FFFFFu) >> 13);
    uint32_t rem = a & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
    return (uint16_t)(sign | h);
}

static uint16_t f32_to_bf16_rne(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    if ((x & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((x >> 16) | 0x40u);
    x += 0x7FFFu + ((x >> 16) & 1u);
    return (uint16_t)(x >> 16);
}

/* out[i] = round_rne(amp * ((z_i >> 40) * 2^-23 - 1)), z_i = mix64(seed + (i+1+offset)*GOLDEN).
 * The fp32 value before rounding is exact (24-bit integer times a power of two).
 * dtype 0 = fp16, 1 = bf16.  amp must be a power of two to keep the pre-rounding value exact. */
int f3si_fill_values(uint16_t* out, int64_t count, int64_t offset, uint64_t seed, int32_t dtype, float amp) {
    if (!out || count < 0 || (dtype != 0 && dtype != 1)) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        uint64_t z = rng_at(seed, (uint64_t)(i + offset));
        float v = ((float)(uint32_t)(z >> 40) * (1.0f / 8388608.0f) - 1.0f) * amp;
        out[i] = dtype == 0 ? f32_to_f16_rne(v) : f32_to_bf16_rne(v);
    }
    return 0;
}

/* exposed for the generator's own tests (checked against numpy's RNE casts) */
void f3si_round_f32(const float* in, uint16_t* out, int64_t count, int32_t dtype) {
    for (int64_t i = 0; i < count; ++i) out[i] = dtype == 0 ? f32_to_f16_rne(in[i]) : f32_to_bf16_rne(in[i]);
}

/* ------------------------------------------------------------------------- */
/* sorting helper: LSD radix sort of uint64 keys with 16-bit digits           */
/* ------------------------------------------------------------------------- */

static int radix_sort_u64(uint64_t* keys, int64_t n) {
    if (n <= 1) return 0;
    uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
    if (!tmp || !cnt) { free(tmp); free(cnt); return 1; }
    uint64_t all_or = 0, all_and = ~0ULL;
    for (int64_t i = 0; i < n; ++i) { all_or |= keys[i]; all_and &= keys[i]; }
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    for (int pass = 0; pass < 4; ++pass) {
        int sh = 16 * pass;
        if ((((all_or ^ all_and) >> sh) & 0xFFFFu) == 0) continue; /* digit constant */
        memset(cnt, 0, 65536 * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> sh) & 0xFFFFu]++;
        int64_t s = 0;
        for (int b = 0; b < 65536; ++b) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> sh) & 0xFFFFu]++] = src[i];
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != keys) memcpy(keys, src, (size_t)n * sizeof(uint64_t));
    free(tmp);
    free(cnt);
    return 0;
}

static int64_t unique_sorted(uint64_t* k, int64_t n) {
    if (n == 0) return 0;
    int64_t m = 1;
    for (int64_t i = 1; i < n; ++i)
        if (k[i] != k[m - 1]) k[m++] = k[i];
    return m;
}

/* ------------------------------------------------------------------------- */
/* alias tables for weighted node sampling                                   */
/* ------------------------------------------------------------------------- */

typedef struct { int64_t n; double* prob; int32_t* alias; int32_t base; } alias_t;

static int alias_build(alias_t* t, const double* w, int64_t n, int32_t base) {
    t->n = n; t->base = base;
    t->prob = (double*)malloc((size_t)n * sizeof(double));
    t->alias = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* small = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* large = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    if (!t->prob || !t->alias || !small || !large) { free(small); free(large); return 1; }
    double sum = 0;
    for (int64_t i = 0; i < n; ++i) sum += w[i];
    int64_t ns = 0, nl = 0;
    for (int64_t i = 0; i < n; ++i) {
        t->prob[i] = w[i] * (double)n / sum;
        t->alias[i] = (int32_t)i;
        if (t->prob[i] < 1.0) small[ns++] = (int32_t)i; else large[nl++] = (int32_t)i;
    }
    while (ns > 0 && nl > 0) {
        int32_t s = small[--ns], l = large[nl - 1];
        t->alias[s] = l;
        t->prob[l] -= 1.0 - t->prob[s];
        if (t->prob[l] < 1.0) { nl--; small[ns++] = l; }
    }
    while (nl > 0) t->prob[large[--nl]] = 1.0;
    while (ns > 0) t->prob[small[--ns]] = 1.0;
    free(small);
    free(large);
    return 0;
}
static void alias_free(alias_t* t) { free(t->prob); free(t->alias); }
static inline int32_t alias_draw(const alias_t* t, uint64_t z) {
    int64_t i = (int64_t)((z >> 32) % (uint64_t)t->n);
    double u = (double)(uint32_t)z * (1.0 / 4294967296.0);
    return t->base + (u < t->prob[i] ? (int32_t)i : t->alias[i]);
}

/* power-law expected-degree weights w_i = (i + i0)^(-1/(gamma-1)), with i0 chosen so that
 * the largest weight carries `max_deg` of a total degree mass `total_deg` (Chung-Lu). */
static void powerlaw_weights(double* w, int64_t n, double gamma, double max_deg, double total_deg) {
    double a = 1.0 / (gamma - 1.0);
    double lo = 0.0, hi = (double)n * 4.0;
    for (int it = 0; it < 100; ++it) {
        double i0 = 0.5 * (lo + hi), s = 0;
        for (int64_t i = 0; i < n; i += (n > 200000 ? 7 : 1)) s += pow((double)i + i0 + 1.0, -a) * (n > 200000 ? 7.0 : 1.0);
        double top = total_deg * pow(i0 + 1.0, -a) / s;
        if (top > max_deg) lo = i0; else hi = i0;
    }
    double i0 = 0.5 * (lo + hi);
    for (int64_t i = 0; i < n; ++i) w[i] = pow((double)i + i0 + 1.0, -a);
}

/* ------------------------------------------------------------------------- */
/* CSR assembly from sorted unique (row<<32 | col) keys                       */
/* ------------------------------------------------------------------------- */

static int keys_to_csr(const uint64_t* k, int64_t m, int32_t n_rows, int32_t** row_ptr, int32_t** col_idx) {
    *row_ptr = (int32_t*)calloc((size_t)n_rows + 1, sizeof(int32_t));
    *col_idx = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    if (!*row_ptr || !*col_idx) return 1;
    for (int64_t i = 0; i < m; ++i) { (*row_ptr)[(k[i] >> 32) + 1]++; (*col_idx)[i] = (int32_t)(k[i] & 0xFFFFFFFFu); }
    for (int32_t r = 0; r < n_rows; ++r) (*row_ptr)[r + 1] += (*row_ptr)[r];
    return 0;
}

/* random permutation of 0..n-1 (Fisher-Yates driven by the counter stream) */
static int32_t* make_perm(int32_t n, uint64_t seed) {
    int32_t* p = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    if (!p) return NULL;
    for (int32_t i = 0; i < n; ++i) p[i] = i;
    for (int32_t i = n - 1; i > 0; --i) {
        int32_t j = (int32_t)(rng_at(seed, (uint64_t)i) % (uint64_t)(i + 1));
        int32_t t = p[i]; p[i] = p[j]; p[j] = t;
    }
    return p;
}

/* Keep exactly `target` of the m unique keys: a seeded uniformly random subset
 * (rank by hash, keep the smallest), re-sorted.  Returns the kept count. */
static int64_t subsample_keys(uint64_t* k, int64_t m, int64_t target, uint64_t seed) {
    if (m <= target) return m;
    uint64_t* hk = (uint64_t*)malloc((size_t)m * sizeof(uint64_t));
    if (!hk) return -1;
    /* threshold selection: the target-th smallest hash, found by sorting a copy of the hashes */
    for (int64_t i = 0; i < m; ++i) hk[i] = mix64(k[i] ^ seed);
    uint64_t* hs = (uint64_t*)malloc((size_t)m * sizeof(uint64_t));
    if (!hs) { free(hk); return -1; }
    memcpy(hs, hk, (size_t)m * sizeof(uint64_t));
    radix_sort_u64(hs, m);
    uint64_t thr = hs[target - 1];
    free(hs);
    int64_t w = 0;
    for (int64_t i = 0; i < m && w < target; ++i)
        if (hk[i] <= thr) k[w++] = k[i];
    free(hk);
    return w;
}

/* ------------------------------------------------------------------------- */
/* Chung-Lu graphs (Cora-, products- and arxiv-shaped)                        */
/* ------------------------------------------------------------------------- */

/*
 * n nodes, exactly `n_pairs` unique pairs (undirected: unordered {u,v}, u!=v;
 * directed: ordered (u,v), u!=v).  Endpoints are drawn with probability proportional
 * to power-law weights (out: gamma/max_deg, in: gamma_in/max_deg_in for directed).
 * symmetrize (undirected only) emits both directions; self_loops adds (i,i);
 * permute relabels nodes by a seeded random permutation.
 */
int f3si_chung_lu(int32_t n, int64_t n_pairs, int32_t directed, double gamma, double max_deg,
                  double gamma_in, double max_deg_in, int32_t symmetrize, int32_t self_loops,
                  int32_t permute, uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    if (n <= 1 || n_pairs < 0 || !row_ptr || !col_idx || !nnz) return 1;
    double* w = (double*)malloc((size_t)n * sizeof(double));
    if (!w) return 2;
    alias_t ta, tb;
    double mass = directed ? (double)n_pairs : 2.0 * (double)n_pairs;
    powerlaw_weights(w, n, gamma, max_deg, mass);
    if (alias_build(&ta, w, n, 0)) return 2;
    if (directed) {
        powerlaw_weights(w, n, gamma_in, max_deg_in, mass);
        /* in-weights are attached to a seeded shuffle of the nodes so that in- and
         * out-degree ranks are independent */
        int32_t* q = make_perm(n, seed ^ 0xA5A5A5A5ULL);
        double* w2 = (double*)malloc((size_t)n * sizeof(double));
        for (int32_t i = 0; i < n; ++i) w2[q[i]] = w[i];
        if (alias_build(&tb, w2, n, 0)) return 2;
        free(q);
        free(w2);
    } else {
        tb = ta;
    }
    free(w);

    int64_t cap = n_pairs + n_pairs / 4 + 1024, m = 0;
    uint64_t* keys = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    if (!keys) return 2;
    uint64_t draw = 0;
    for (int round = 0; round < 64 && m < n_pairs; ++round) {
        int64_t want = (n_pairs - m) + (n_pairs - m) / 8 + 64;
        if (m + want > cap) {
            cap = m + want;
            keys = (uint64_t*)realloc(keys, (size_t)cap * sizeof(uint64_t));
            if (!keys) return 2;
        }
        uint64_t base = draw;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < want; ++i) {
            uint64_t z1 = rng_at(seed, 2 * (base + (uint64_t)i));
            uint64_t z2 = rng_at(seed, 2 * (base + (uint64_t)i) + 1);
            uint64_t u = (uint64_t)alias_draw(&ta, z1), v = (uint64_t)alias_draw(&tb, z2);
            if (!directed && u > v) { uint64_t t = u; u = v; v = t; }
            keys[m + i] = (u == v) ? ~0ULL : ((u << 32) | v);
        }
        draw += (uint64_t)want;
        m += want;
        if (radix_sort_u64(keys, m)) return 2;
        m = unique_sorted(keys, m);
        if (m > 0 && keys[m - 1] == ~0ULL) m--; /* drop the self-pair sentinel */
    }
    alias_free(&ta);
    if (directed) alias_free(&tb);
    m = subsample_keys(keys, m, n_pairs, seed ^ 0x5151ULL);
    if (m < 0) return 2;

    int32_t* perm = permute ? make_perm(n, seed ^ 0x7E7EULL) : NULL;
    int64_t total = m * ((!directed && symmetrize) ? 2 : 1) + (self_loops ? n : 0);
    uint64_t* out = (uint64_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint64_t));
    if (!out) return 2;
    int64_t o = 0;
    for (int64_t i = 0; i < m; ++i) {
        uint64_t u = keys[i] >> 32, v = keys[i] & 0xFFFFFFFFu;
        if (perm) { u = (uint64_t)perm[u]; v = (uint64_t)perm[v]; }
        out[o++] = (u << 32) | v;
        if (!directed && symmetrize) out[o++] = (v << 32) | u;
    }
    if (self_loops)
        for (int64_t i = 0; i < n; ++i) out[o++] = ((uint64_t)i << 32) | (uint64_t)i;
    free(keys);
    free(perm);
    if (radix_sort_u64(out, o)) return 2;
    o = unique_sorted(out, o);
    int rc = keys_to_csr(out, o, n, row_ptr, col_idx);
    free(out);
    *nnz = o;
    return rc ? 2 : 0;
}

/* ------------------------------------------------------------------------- */
/* Degree-corrected block model (Reddit-shaped)                              */
/* ------------------------------------------------------------------------- */

/*
 * Contiguous-ID communities of `comm_size` nodes.  Each undirected pair draws its first
 * endpoint u by power-law weight; with probability `mu` the second endpoint is drawn by
 * weight inside u's community, otherwise globally.  Symmetric, no self-loops, IDs not
 * permuted (communities stay contiguous, which is what gives Reddit its shared columns).
 */
static int dcsbm_core(int32_t n, int64_t n_pairs, int32_t comm_size, double mu, const double* mu_node, double* wn,
                      uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz);

int f3si_dcsbm(int32_t n, int64_t n_pairs, int32_t comm_size, double mu, double gamma, double max_deg,
               uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    if (n <= 1 || comm_size < 2 || n_pairs < 0) return 1;
    double* w = (double*)malloc((size_t)n * sizeof(double));
    if (!w) return 2;
    powerlaw_weights(w, n, gamma, max_deg, 2.0 * (double)n_pairs);
    /* spread heavy nodes over communities: weight rank -> node via seeded permutation */
    int32_t* q = make_perm(n, seed ^ 0x3C3CULL);
    double* wn = (double*)malloc((size_t)n * sizeof(double));
    for (int32_t i = 0; i < n; ++i) wn[q[i]] = w[i];
    free(q);
    free(w);
    return dcsbm_core(n, n_pairs, comm_size, mu, NULL, wn, seed, row_ptr, col_idx, nnz);
}

/*
 * Same block model with caller-given node weights w[n] (expected-degree shape; only ratios
 * matter) and a local fraction per first endpoint (mu_node[n]).  The Reddit-shaped workload passes weights that are constant-ish within each
 * 16-row window and drawn per window from the paper's TCB/RW decile table,
 * which is what gives the row windows their long-tailed widths.
 */
int f3si_dcsbm_w(int32_t n, int64_t n_pairs, int32_t comm_size, const double* mu_node, const double* w,
                 uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    if (n <= 1 || comm_size < 2 || n_pairs < 0 || !w || !mu_node) return 1;
    double* wn = (double*)malloc((size_t)n * sizeof(double));
    if (!wn) return 2;
    memcpy(wn, w, (size_t)n * sizeof(double));
    return dcsbm_core(n, n_pairs, comm_size, 0.0, mu_node, wn, seed, row_ptr, col_idx, nnz);
}

/* takes ownership of wn; mu_node (optional) gives each first endpoint its own local fraction */
static int dcsbm_core(int32_t n, int64_t n_pairs, int32_t comm_size, double mu, const double* mu_node, double* wn,
                      uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    int32_t n_comm = (n + comm_size - 1) / comm_size;
    alias_t glob;
    if (alias_build(&glob, wn, n, 0)) return 2;
    alias_t* loc = (alias_t*)malloc((size_t)n_comm * sizeof(alias_t));
    for (int32_t c = 0; c < n_comm; ++c) {
        int32_t b = c * comm_size, e = b + comm_size < n ? b + comm_size : n;
        if (alias_build(&loc[c], wn + b, e - b, b)) return 2;
    }
    free(wn);
    int64_t cap = n_pairs + n_pairs / 4 + 1024, m = 0;
    uint64_t* keys = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    uint64_t draw = 0;
    for (int round = 0; round < 64 && m < n_pairs; ++round) {
        int64_t want = (n_pairs - m) + (n_pairs - m) / 4 + 64;
        if (m + want > cap) { cap = m + want; keys = (uint64_t*)realloc(keys, (size_t)cap * sizeof(uint64_t)); }
        if (!keys) return 2;
        uint64_t base = draw;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < want; ++i) {
            uint64_t z1 = rng_at(seed, 3 * (base + (uint64_t)i));
            uint64_t z2 = rng_at(seed, 3 * (base + (uint64_t)i) + 1);
            uint64_t z3 = rng_at(seed, 3 * (base + (uint64_t)i) + 2);
            uint64_t u = (uint64_t)alias_draw(&glob, z1);
            uint64_t v = (u01(z3) < (mu_node ? mu_node[u] : mu)) ? (uint64_t)alias_draw(&loc[u / (uint64_t)comm_size], z2)
                                         : (uint64_t)alias_draw(&glob, z2);
            if (u > v) { uint64_t t = u; u = v; v = t; }
            keys[m + i] = (u == v) ? ~0ULL : ((u << 32) | v);
        }
        draw += (uint64_t)want;
        m += want;
        radix_sort_u64(keys, m);
        m = unique_sorted(keys, m);
        if (m > 0 && keys[m - 1] == ~0ULL) m--;
    }
    alias_free(&glob);
    for (int32_t c = 0; c < n_comm; ++c) alias_free(&loc[c]);
    free(loc);
    m = subsample_keys(keys, m, n_pairs, seed ^ 0x5151ULL);
    uint64_t* out = (uint64_t*)malloc((size_t)(2 * m + 1) * sizeof(uint64_t));
    int64_t o = 0;
    for (int64_t i = 0; i < m; ++i) {
        uint64_t u = keys[i] >> 32, v = keys[i] & 0xFFFFFFFFu;
        out[o++] = (u << 32) | v;
        out[o++] = (v << 32) | u;
    }
    free(keys);
    radix_sort_u64(out, o);
    o = unique_sorted(out, o);
    int rc = keys_to_csr(out, o, n, row_ptr, col_idx);
    free(out);
    *nnz = o;
    return rc ? 2 : 0;
}

/* ------------------------------------------------------------------------- */
/* Row-window construction (Reddit-shaped: long-tailed window widths)         */
/* ------------------------------------------------------------------------- */

/*
 * Builds A window by window so that the 16x8 plan statistics of Tab.datasets / Tab.tcb_deciles
 * hold by construction.  Window k (rows 16k .. 16k+15) gets exactly
 * U_k = min(8 * tcb[k], n) distinct columns: each draw is, with probability mu, a node of the
 * window's own community (contiguous IDs, comm_size nodes, uniform) and otherwise a node drawn
 * by a global power-law popularity (exponent gamma, hubs at seeded random IDs); every column is
 * then hit by m distinct rows of the window, m = 1 + Poisson(ratio[k] / 8 - 1) clipped to the
 * window's rows, so that nnz_k / tcb_k has mean ratio[k].  Not symmetric (the statistics are
 * those of the row windows).  Rows sorted, no duplicates.  Windows are independent: the
 * result does not depend on the thread count.
 */
static inline uint64_t hash_probe(uint64_t x) { return mix64(x ^ 0x6A09E667F3BCC909ULL); }

int f3si_windows(int32_t n, const int32_t* tcb, const double* ratio, int32_t comm_size, double mu, double gamma,
                 uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    if (n < 1 || comm_size < 1 || !tcb || !ratio || !row_ptr || !col_idx || !nnz) return 1;
    const int32_t R = (n + 15) / 16;
    double* w = (double*)malloc((size_t)n * sizeof(double));
    if (!w) return 2;
    double a = 1.0 / (gamma - 1.0);
    for (int32_t i = 0; i < n; ++i) w[i] = pow((double)i + 10.0, -a);
    int32_t* q = make_perm(n, seed ^ 0x1D1DULL);
    double* wn = (double*)malloc((size_t)n * sizeof(double));
    for (int32_t i = 0; i < n; ++i) wn[q[i]] = w[i];
    free(q);
    free(w);
    alias_t glob;
    if (alias_build(&glob, wn, n, 0)) return 2;
    free(wn);
    /* per-window entry counts are random: each window fills its own buffer */
    uint64_t** bufs = (uint64_t**)calloc((size_t)R, sizeof(uint64_t*));
    int64_t* cnt = (int64_t*)calloc((size_t)R, sizeof(int64_t));
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 16)
    for (int32_t k = 0; k < R; ++k) {
        const int32_t r0 = 16 * k, nr = (r0 + 16 <= n) ? 16 : n - r0;
        int64_t U = (int64_t)8 * tcb[k];
        if (U > n) U = n;
        if (U < 0) U = 0;
        int64_t tsize = 64;
        while (tsize < 2 * U) tsize <<= 1;
        int32_t* table = (int32_t*)malloc((size_t)tsize * sizeof(int32_t));
        int32_t* chosen = (int32_t*)malloc((size_t)(U > 0 ? U : 1) * sizeof(int32_t));
        uint64_t* out = (uint64_t*)malloc((size_t)(U * nr > 0 ? U * nr : 1) * sizeof(uint64_t));
        if (!table || !chosen || !out) { fail = 1; free(table); free(chosen); free(out); continue; }
        for (int64_t t = 0; t < tsize; ++t) table[t] = -1;
        const int32_t c0 = (r0 / comm_size) * comm_size;
        const int32_t cs = (c0 + comm_size <= n) ? comm_size : n - c0;
        uint64_t ctr = 0, wseed = mix64(seed + (uint64_t)k * GOLDEN);
        int64_t got = 0, local_got = 0, tries = 0;
        while (got < U && tries < 64 * U + 4096) {
            ++tries;
            const uint64_t z1 = rng_at(wseed, ctr++), z2 = rng_at(wseed, ctr++);
            int32_t c;
            /* local draws stop once the community is nearly exhausted */
            if (u01(z1) < mu && local_got < (int64_t)cs * 7 / 8) c = c0 + (int32_t)(z2 % (uint64_t)cs);
            else c = alias_draw(&glob, z2);
            uint64_t hslot = hash_probe((uint64_t)c) & (uint64_t)(tsize - 1);
            int dup = 0;
            while (table[hslot] >= 0) {
                if (table[hslot] == c) { dup = 1; break; }
                hslot = (hslot + 1) & (uint64_t)(tsize - 1);
            }
            if (dup) continue;
            table[hslot] = c;
            chosen[got++] = c;
            if (c >= c0 && c < c0 + cs) ++local_got;
        }
        /* rows hitting each column: m = 1 + Poisson(lambda), distinct rows (partial shuffle) */
        const double lam = ratio[k] / 8.0 - 1.0 > 0.0 ? ratio[k] / 8.0 - 1.0 : 0.0;
        const double el = exp(-lam);
        int64_t o = 0;
        for (int64_t u = 0; u < got; ++u) {
            int32_t m = 1;
            double prod = u01(rng_at(wseed, ctr++));
            while (prod > el && m < nr) { ++m; prod *= u01(rng_at(wseed, ctr++)); }
            int32_t perm[16];
            for (int32_t i = 0; i < nr; ++i) perm[i] = i;
            for (int32_t i = 0; i < m; ++i) {
                int32_t j = i + (int32_t)(rng_at(wseed, ctr++) % (uint64_t)(nr - i));
                int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
                out[o++] = ((uint64_t)(r0 + perm[i]) << 32) | (uint64_t)(uint32_t)chosen[u];
            }
        }
        free(table);
        free(chosen);
        bufs[k] = out;
        cnt[k] = o;
    }
    alias_free(&glob);
    if (fail) return 2;
    int64_t total = 0;
    for (int32_t k = 0; k < R; ++k) total += cnt[k];
    uint64_t* all = (uint64_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint64_t));
    if (!all) return 2;
    int64_t o = 0;
    for (int32_t k = 0; k < R; ++k) {
        memcpy(all + o, bufs[k], (size_t)cnt[k] * sizeof(uint64_t));
        o += cnt[k];
        free(bufs[k]);
    }
    free(bufs);
    free(cnt);
    if (radix_sort_u64(all, o)) return 2;
    o = unique_sorted(all, o);
    int rc = keys_to_csr(all, o, n, row_ptr, col_idx);
    free(all);
    *nnz = o;
    return rc ? 2 : 0;
}

/* ------------------------------------------------------------------------- */
/* Batched molecule-like graphs (ZINC/LRGB-shaped), block-diagonal union      */
/* ------------------------------------------------------------------------- */

/*
 * n_graphs graphs with node counts uniform in [n_min, n_max].  Each graph is a random
 * tree with local attachment (node t's parent lies within the previous <=4 IDs) plus
 * about n_g/15 ring-closing edges between IDs 2..6 apart.  IDs are contiguous per graph
 * (batching = block-diagonal union).  Symmetric; optional self-loops.
 * graph_ptr (n_graphs+1) receives the first node of each graph.
 */
int f3si_molecules(int32_t n_graphs, int32_t n_min, int32_t n_max, int32_t self_loops, uint64_t seed,
                   int32_t** row_ptr, int32_t** col_idx, int64_t* nnz, int32_t* n_out, int32_t** graph_ptr) {
    if (n_graphs < 1 || n_min < 2 || n_max < n_min) return 1;
    int32_t* gp = (int32_t*)malloc((size_t)(n_graphs + 1) * sizeof(int32_t));
    gp[0] = 0;
    for (int32_t g = 0; g < n_graphs; ++g)
        gp[g + 1] = gp[g] + n_min + (int32_t)(rng_at(seed, (uint64_t)g) % (uint64_t)(n_max - n_min + 1));
    int32_t n = gp[n_graphs];
    int64_t cap = (int64_t)n * 3 + 16, o = 0;
    uint64_t* out = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
    uint64_t s2 = seed ^ 0xBEEFULL;
    for (int32_t g = 0; g < n_graphs; ++g) {
        int32_t b = gp[g], ng = gp[g + 1] - gp[g];
        uint64_t ctr = (uint64_t)b * 4;
        for (int32_t t = 1; t < ng; ++t) {
            int32_t span = t < 4 ? t : 4;
            int32_t p = t - 1 - (int32_t)(rng_at(s2, ctr++) % (uint64_t)span);
            uint64_t u = (uint64_t)(b + p), v = (uint64_t)(b + t);
            out[o++] = (u << 32) | v;
            out[o++] = (v << 32) | u;
        }
        int32_t rings = ng / 15;
        for (int32_t r = 0; r < rings; ++r) {
            int32_t a = (int32_t)(rng_at(s2, ctr++) % (uint64_t)(ng - 2));
            int32_t c = a + 2 + (int32_t)(rng_at(s2, ctr++) % 5ULL);
            if (c >= ng) c = ng - 1;
            if (c == a) continue;
            uint64_t u = (uint64_t)(b + a), v = (uint64_t)(b + c);
            if (o + 2 > cap) { cap *= 2; out = (uint64_t*)realloc(out, (size_t)cap * sizeof(uint64_t)); }
            out[o++] = (u << 32) | v;
            out[o++] = (v << 32) | u;
        }
        if (o + 2 * 16 > cap) { cap *= 2; out = (uint64_t*)realloc(out, (size_t)cap * sizeof(uint64_t)); }
    }
    if (self_loops) {
        out = (uint64_t*)realloc(out, (size_t)(o + n) * sizeof(uint64_t));
        for (int64_t i = 0; i < n; ++i) out[o++] = ((uint64_t)i << 32) | (uint64_t)i;
    }
    radix_sort_u64(out, o);
    o = unique_sorted(out, o);
    int rc = keys_to_csr(out, o, n, row_ptr, col_idx);
    free(out);
    *nnz = o;
    *n_out = n;
    *graph_ptr = gp;
    return rc ? 2 : 0;
}

/* Uniform random CSR (tests): each row gets a degree in [deg_min, deg_max] with columns drawn
 * uniformly from [0, n_cols); duplicates kept or merged per `keep_dups`, rows optionally unsorted. */
int f3si_random_csr(int32_t n_rows, int32_t n_cols, int32_t deg_min, int32_t deg_max, int32_t keep_dups,
                    int32_t shuffle_rows, uint64_t seed, int32_t** row_ptr, int32_t** col_idx, int64_t* nnz) {
    if (n_rows < 0 || n_cols < 1 || deg_min < 0 || deg_max < deg_min) return 1;
    int32_t* rp = (int32_t*)malloc((size_t)(n_rows + 1) * sizeof(int32_t));
    rp[0] = 0;
    for (int32_t r = 0; r < n_rows; ++r)
        rp[r + 1] = rp[r] + deg_min + (int32_t)(rng_at(seed, (uint64_t)r) % (uint64_t)(deg_max - deg_min + 1));
    int64_t m = rp[n_rows];
    int32_t* ci = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    uint64_t s2 = seed ^ 0x1234ULL;
    for (int64_t i = 0; i < m; ++i) ci[i] = (int32_t)(rng_at(s2, (uint64_t)i) % (uint64_t)n_cols);
    /* rows are left in draw order (unsorted, duplicates possible) unless asked otherwise */
    if (!shuffle_rows || !keep_dups) {
        int32_t* ri = (int32_t*)malloc((size_t)(n_rows + 1) * sizeof(int32_t));
        int64_t w = 0;
        ri[0] = 0;
        for (int32_t r = 0; r < n_rows; ++r) {
            int64_t b = rp[r], e = rp[r + 1];
            /* insertion sort: rows are short in tests */
            for (int64_t i = b + 1; i < e; ++i) {
                int32_t x = ci[i];
                int64_t j = i - 1;
                while (j >= b && ci[j] > x) { ci[j + 1] = ci[j]; --j; }
                ci[j + 1] = x;
            }
            for (int64_t i = b; i < e; ++i)
                if (keep_dups || i == b || ci[i] != ci[i - 1]) ci[w++] = ci[i];
            ri[r + 1] = (int32_t)w;
        }
        free(rp);
        rp = ri;
        m = w;
    }
    *row_ptr = rp;
    *col_idx = ci;
    *nnz = m;
    return 0;
}

void f3si_free(void* p) { free(p); }
