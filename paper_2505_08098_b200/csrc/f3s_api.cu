// f3s_api.cu — the C ABI of include/f3s.h: argument validation, status codes, plan
// ownership, host-buffer end-to-end call, row partitioner.  No C++ exception crosses it.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <new>
#include <mutex>
#include <string>

#include "internal.h"

namespace f3s {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            cudaMemPool_t np = nullptr;
            if ((e = cudaMemPoolCreate(&np, &props)) != cudaSuccess) return e;
            // keep freed scratch reserved across synchronisations: the backward's per-call workspace
            // (a few GB) would otherwise be unmapped at every sync and mapped again by the next call
            // (measured: 9-170 ms per call instead of 3.7 ms, tools/bwd_percall.py)
            uint64_t keep = ~uint64_t(0);
            if ((e = cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
            pools[dev] = np;
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(ptr, bytes ? bytes : 16, pool, stream);
}

cudaError_t scratch_free(void* ptr, cudaStream_t stream) { return ptr ? cudaFreeAsync(ptr, stream) : cudaSuccess; }

f3s_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    (void)cudaGetLastError();  // clear a sticky-free error so later calls are not poisoned
    return e == cudaErrorMemoryAllocation ? F3S_ERR_OUT_OF_MEMORY : F3S_ERR_CUDA;
}

static f3s_status check_attention_args(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O,
                                       float scale, int32_t heads, int32_t d, f3s_dtype dtype, bool device) {
    if (!plan) { set_error("plan is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (heads < 1) { set_error("heads must be >= 1"); return F3S_ERR_INVALID_VALUE; }
    if (!std::isfinite(scale)) { set_error("scale must be finite"); return F3S_ERR_INVALID_VALUE; }
    if (dtype != F3S_FP16 && dtype != F3S_BF16 && dtype != F3S_E4M3) {
        set_error("dtype must be F3S_FP16, F3S_BF16 or F3S_E4M3");
        return F3S_ERR_INVALID_VALUE;
    }
    const Plan& p = *reinterpret_cast<const Plan*>(plan);
    if (p.n_rows > 0 && (!Q || !O)) { set_error("Q/O is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (p.n_cols > 0 && (!K || !V)) { set_error("K/V is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (d != 64 && d != 128) { set_error("d must be 64 or 128"); return F3S_ERR_UNSUPPORTED; }
    if ((int64_t)heads * d > (int64_t)1 << 24) { set_error("heads*d too large"); return F3S_ERR_UNSUPPORTED; }
    if ((int64_t)p.num_rw * heads > 0x7FFFFFFFLL) { set_error("num_rw*heads >= 2^31"); return F3S_ERR_UNSUPPORTED; }
    if (device) {
        auto mis = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) != 0; };
        if (mis(Q) || mis(K) || mis(V) || mis(O)) { set_error("Q/K/V/O must be 16-byte aligned"); return F3S_ERR_UNSUPPORTED; }
        if (O && (O == Q || O == K || O == V)) { set_error("O aliases an input"); return F3S_ERR_INVALID_VALUE; }
    }
    return F3S_OK;
}

static f3s_status run_attention(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                                int32_t heads, int32_t d, f3s_dtype dtype, f3s_variant variant, cudaStream_t stream,
                                uint64_t* trace = nullptr, int32_t trace_chunks = 0, int32_t grid = 0,
                                int64_t kv_ld = 0, int64_t q_ld = 0) {
    f3s_status st = check_attention_args(plan, Q, K, V, O, scale, heads, d, dtype, true);
    if (st != F3S_OK) return st;
    if (q_ld != 0 && (q_ld < (int64_t)heads * d || (q_ld * (dtype == F3S_E4M3 ? 1 : 2)) % 16 != 0)) {
        set_error("q_row_stride must be >= heads * d and a multiple of 16 bytes");
        return F3S_ERR_INVALID_VALUE;
    }
    if (q_ld != 0 && variant == F3S_VARIANT_SIMT) { set_error("q_row_stride: tcgen05 variants only"); return F3S_ERR_UNSUPPORTED; }
    if (kv_ld != 0) {
        if (kv_ld < (int64_t)heads * d) { set_error("kv_row_stride < heads * d"); return F3S_ERR_INVALID_VALUE; }
        if ((kv_ld * (dtype == F3S_E4M3 ? 1 : 2)) % 16 != 0) {
            set_error("kv_row_stride must be a multiple of 16 bytes");
            return F3S_ERR_UNSUPPORTED;
        }
        if (variant == F3S_VARIANT_SIMT) { set_error("kv_row_stride: tcgen05 variants only"); return F3S_ERR_UNSUPPORTED; }
    }
    AttnArgs a{reinterpret_cast<const Plan*>(plan), Q, K, V, O, scale, heads, d, dtype,
               variant != F3S_VARIANT_NO_REORDER, stream};
    a.kv_ld = kv_ld;
    a.q_ld = q_ld;
    a.trace = trace_chunks < 0 ? nullptr : trace;
    a.trace_chunks = trace_chunks < 0 ? 0 : trace_chunks;
    a.expt = trace_chunks < 0 ? -trace_chunks : 0;
    a.grid_override = grid;
    a.one_head = variant == F3S_VARIANT_ONE_HEAD;
    if (a.plan->n_rows == 0) return F3S_OK;
    if (dtype == F3S_E4M3 && (variant == F3S_VARIANT_SIMT || variant == F3S_VARIANT_ONE_HEAD)) {
        set_error("F3S_E4M3: DEFAULT and NO_REORDER variants only");
        return F3S_ERR_UNSUPPORTED;
    }
    // launch on the plan's device whatever the calling thread's current device is
    DeviceScope scope;
    F3S_CUDA_TRY(scope.enter(a.plan->device));
    switch (variant) {
        case F3S_VARIANT_DEFAULT:
        case F3S_VARIANT_NO_REORDER:
        case F3S_VARIANT_ONE_HEAD: return launch_attention_sm100(a);
        case F3S_VARIANT_SIMT: return launch_attention_simt(a);
        default: set_error("unknown variant"); return F3S_ERR_INVALID_VALUE;
    }
}

}  // namespace f3s

using namespace f3s;

extern "C" {

f3s_status f3s_plan(const int32_t* row_ptr, const int32_t* col_idx, int32_t n, cudaStream_t stream, f3s_plan_t* out) {
    if (!out) { set_error("out is NULL"); return F3S_ERR_INVALID_VALUE; }
    *out = nullptr;
    try {
        Plan* p = nullptr;
        f3s_status st = build_plan(row_ptr, col_idx, n, n, true, stream, &p);
        if (st == F3S_OK) *out = reinterpret_cast<f3s_plan_t>(p);
        return st;
    } catch (const std::bad_alloc&) {
        return F3S_ERR_OUT_OF_MEMORY;
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_plan_rows(const int32_t* row_ptr, const int32_t* col_idx, int32_t n_rows, int32_t n_cols,
                         cudaStream_t stream, f3s_plan_t* out) {
    if (!out) { set_error("out is NULL"); return F3S_ERR_INVALID_VALUE; }
    *out = nullptr;
    try {
        Plan* p = nullptr;
        f3s_status st = build_plan(row_ptr, col_idx, n_rows, n_cols, false, stream, &p);
        if (st == F3S_OK) *out = reinterpret_cast<f3s_plan_t>(p);
        return st;
    } catch (const std::bad_alloc&) {
        return F3S_ERR_OUT_OF_MEMORY;
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_plan_destroy(f3s_plan_t plan) {
    if (!plan) return F3S_OK;
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (p->tplan) f3s_plan_destroy(reinterpret_cast<f3s_plan_t>(p->tplan));
    cudaFree(p->rw_ptr);
    cudaFree(p->cols);
    cudaFree(p->masks);
    cudaFree(p->rw_order);
    cudaFree(p->rw_natural);
    cudaFree(p->kcols);
    cudaFree(p->kmasks);
    cudaFree(p->meta_lpt);
    cudaFree(p->meta_nat);
    cudaFree(p->meta_sub);
    cudaFree(p->ginfo);
    cudaFree(p->col_ptr);
    cudaFree(p->col_rows);
    cudaFree(p->col_lists);
    cudaFree(p->heavy_rows);
    cudaFree(p->heavy_row_flag);
    for (auto& st : p->staging) cudaFree(st.ptr);
    delete p;
    return F3S_OK;
}

f3s_status f3s_plan_set_split(f3s_plan_t plan, int32_t max_chunks) {
    if (!plan) { set_error("plan is NULL"); return F3S_ERR_INVALID_VALUE; }
    try {
        Plan* p = reinterpret_cast<Plan*>(plan);
        DeviceScope scope;
        F3S_CUDA_TRY(scope.enter(p->device));
        return build_split(p, max_chunks);
    } catch (const std::bad_alloc&) {
        return F3S_ERR_OUT_OF_MEMORY;
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

int32_t f3s_default_split_chunks(int64_t total_chunks, int32_t num_sms) {
    return default_split_chunks(total_chunks, num_sms);
}

f3s_status f3s_plan_get_info(f3s_plan_t plan, f3s_plan_info* info) {
    if (!plan || !info) { set_error("plan/info is NULL"); return F3S_ERR_INVALID_VALUE; }
    const Plan& p = *reinterpret_cast<const Plan*>(plan);
    std::memset(info, 0, sizeof(*info));
    info->n_rows = p.n_rows;
    info->n_cols = p.n_cols;
    info->num_rw = p.num_rw;
    info->max_width = p.max_width;
    info->nnz = p.nnz;
    info->total_cols = p.total_cols;
    info->total_tcb8 = p.total_tcb8;
    info->device_bytes = p.device_bytes;
    info->build_ms = p.build_ms;
    info->split_chunks = p.split_chunks;
    info->split_groups = p.n_groups;
    info->total_chunks = p.total_chunks;
    return F3S_OK;
}

f3s_status f3s_plan_export(f3s_plan_t plan, int32_t* rw_ptr, int32_t* cols, uint16_t* masks, int32_t* rw_order) {
    if (!plan) { set_error("plan is NULL"); return F3S_ERR_INVALID_VALUE; }
    const Plan& p = *reinterpret_cast<const Plan*>(plan);
    if (rw_ptr) F3S_CUDA_TRY(cudaMemcpy(rw_ptr, p.rw_ptr, sizeof(int32_t) * (p.num_rw + 1), cudaMemcpyDeviceToHost));
    if (cols && p.total_cols) F3S_CUDA_TRY(cudaMemcpy(cols, p.cols, sizeof(int32_t) * p.total_cols, cudaMemcpyDeviceToHost));
    if (masks && p.total_cols) F3S_CUDA_TRY(cudaMemcpy(masks, p.masks, sizeof(uint16_t) * p.total_cols, cudaMemcpyDeviceToHost));
    if (rw_order && p.num_rw) F3S_CUDA_TRY(cudaMemcpy(rw_order, p.rw_order, sizeof(int32_t) * p.num_rw, cudaMemcpyDeviceToHost));
    return F3S_OK;
}

f3s_status f3s_attention(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                         int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    try {
        return run_attention(plan, Q, K, V, O, scale, heads, d, dtype, F3S_VARIANT_DEFAULT, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_backward(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* dO,
                                  float* dQ, float* dK, float* dV, float scale, int32_t heads, int32_t d,
                                  f3s_dtype dtype, cudaStream_t stream) {
    return f3s_attention_backward_ex(plan, Q, K, V, dO, dQ, dK, dV, scale, heads, d, dtype, 0, stream);
}

f3s_status f3s_attention_backward_ex(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* dO,
                                     float* dQ, float* dK, float* dV, float scale, int32_t heads, int32_t d,
                                     f3s_dtype dtype, int32_t variant, cudaStream_t stream) {
    try {
        f3s_status st = check_attention_args(plan, Q, K, V, dQ, scale, heads, d, dtype, true);
        if (st != F3S_OK) return st;
        if (dtype == F3S_E4M3) { set_error("backward: F3S_FP16 or F3S_BF16 only"); return F3S_ERR_UNSUPPORTED; }
        Plan& p = *reinterpret_cast<Plan*>(plan);
        if (p.n_rows > 0 && !dO) { set_error("dO is NULL"); return F3S_ERR_INVALID_VALUE; }
        if (p.n_cols > 0 && (!dK || !dV)) { set_error("dK/dV is NULL"); return F3S_ERR_INVALID_VALUE; }
        if (variant != 0 && variant != 1) { set_error("backward variant must be 0 or 1"); return F3S_ERR_INVALID_VALUE; }
        auto mis = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) != 0; };
        if (mis(dO) || mis(dK) || mis(dV)) { set_error("dO/dK/dV must be 16-byte aligned"); return F3S_ERR_UNSUPPORTED; }
        DeviceScope scope;
        F3S_CUDA_TRY(scope.enter(p.device));
        if (variant == 0 && p.nnz > 0 && p.n_rows > 0)
            return launch_attention_backward_tc(p, Q, K, V, nullptr, nullptr, dO, false, dQ, dK, dV, scale, heads, d,
                                                dtype, stream);
        return launch_attention_backward(p, Q, K, V, dO, dQ, dK, dV, scale, heads, d, dtype, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_fwd(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float* ml,
                             float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    try {
        f3s_status st = check_attention_args(plan, Q, K, V, O, scale, heads, d, dtype, true);
        if (st != F3S_OK) return st;
        const Plan& p = *reinterpret_cast<const Plan*>(plan);
        if (p.n_rows > 0 && !ml) { set_error("ml is NULL"); return F3S_ERR_INVALID_VALUE; }
        if (reinterpret_cast<uintptr_t>(ml) & 7) { set_error("ml must be 8-byte aligned"); return F3S_ERR_UNSUPPORTED; }
        if (p.n_rows == 0) return F3S_OK;
        AttnArgs a{&p, Q, K, V, O, scale, heads, d, dtype, true, stream};
        a.ml_out = ml;
        a.ml_norm = true;
        DeviceScope scope;
        F3S_CUDA_TRY(scope.enter(p.device));
        if (p.nnz == 0 || p.n_cols == 0) {  // every row is empty: O = 0, (m, l) = (floor, 0) (reading c4)
            F3S_CUDA_TRY(cudaMemsetAsync(O, 0, sizeof(float) * (size_t)p.n_rows * heads * d, stream));
            return launch_fill_ml(ml, (int64_t)p.n_rows * heads, stream);
        }
        return launch_attention_sm100(a);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

static f3s_status backward_saved_impl(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* O,
                                      const float* ml, const void* dO, bool dO_lp, void* dQ, void* dK, void* dV,
                                      float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    f3s_status st = check_attention_args(plan, Q, K, V, static_cast<float*>(dQ), scale, heads, d, dtype, true);
    if (st != F3S_OK) return st;
    if (dtype == F3S_E4M3) { set_error("backward: F3S_FP16 or F3S_BF16 only"); return F3S_ERR_UNSUPPORTED; }
    Plan& p = *reinterpret_cast<Plan*>(plan);
    if (p.n_rows > 0 && (!dO || !O || !ml)) { set_error("O/ml/dO is NULL"); return F3S_ERR_INVALID_VALUE; }
    if (p.n_cols > 0 && (!dK || !dV)) { set_error("dK/dV is NULL"); return F3S_ERR_INVALID_VALUE; }
    auto mis = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) != 0; };
    if (mis(dO) || mis(dK) || mis(dV) || mis(O)) { set_error("O/dO/dK/dV must be 16-byte aligned"); return F3S_ERR_UNSUPPORTED; }
    if (reinterpret_cast<uintptr_t>(ml) & 7) { set_error("ml must be 8-byte aligned"); return F3S_ERR_UNSUPPORTED; }
    DeviceScope scope;
    F3S_CUDA_TRY(scope.enter(p.device));
    if (p.nnz > 0 && p.n_rows > 0)
        return launch_attention_backward_tc(p, Q, K, V, O, ml, dO, dO_lp, dQ, dK, dV, scale, heads, d, dtype, stream);
    // every row empty: all gradients are zero
    const size_t es = dO_lp ? 2 : sizeof(float);
    if (p.n_rows > 0) F3S_CUDA_TRY(cudaMemsetAsync(dQ, 0, es * (size_t)p.n_rows * heads * d, stream));
    if (p.n_cols > 0) {
        F3S_CUDA_TRY(cudaMemsetAsync(dK, 0, es * (size_t)p.n_cols * heads * d, stream));
        F3S_CUDA_TRY(cudaMemsetAsync(dV, 0, es * (size_t)p.n_cols * heads * d, stream));
    }
    return F3S_OK;
}

f3s_status f3s_attention_backward_saved(f3s_plan_t plan, const void* Q, const void* K, const void* V, const float* O,
                                        const float* ml, const float* dO, float* dQ, float* dK, float* dV, float scale,
                                        int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    try {
        return backward_saved_impl(plan, Q, K, V, O, ml, dO, false, dQ, dK, dV, scale, heads, d, dtype, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_backward_saved_lp(f3s_plan_t plan, const void* Q, const void* K, const void* V,
                                           const float* O, const float* ml, const void* dO, void* dQ, void* dK,
                                           void* dV, float scale, int32_t heads, int32_t d, f3s_dtype dtype,
                                           cudaStream_t stream) {
    try {
        return backward_saved_impl(plan, Q, K, V, O, ml, dO, true, dQ, dK, dV, scale, heads, d, dtype, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_kv(f3s_plan_t plan, const void* Q, const void* K, const void* V, int64_t kv_row_stride,
                            float* O, float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    try {
        return run_attention(plan, Q, K, V, O, scale, heads, d, dtype, F3S_VARIANT_DEFAULT, stream, nullptr, 0, 0,
                             kv_row_stride);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_strided(f3s_plan_t plan, const void* Q, int64_t q_row_stride, const void* K, const void* V,
                                 int64_t kv_row_stride, float* O, float scale, int32_t heads, int32_t d,
                                 f3s_dtype dtype, cudaStream_t stream) {
    try {
        return run_attention(plan, Q, K, V, O, scale, heads, d, dtype, F3S_VARIANT_DEFAULT, stream, nullptr, 0, 0,
                             kv_row_stride, q_row_stride);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_partial(f3s_plan_t plan, const void* Q, const void* K, const void* V, int64_t kv_row_stride,
                                 float* O_part, float* ml_part, float scale, int32_t heads, int32_t d, f3s_dtype dtype,
                                 int32_t max_ctas, cudaStream_t stream) {
    try {
        f3s_status st = check_attention_args(plan, Q, K, V, O_part, scale, heads, d, dtype, true);
        if (st != F3S_OK) return st;
        const Plan& p = *reinterpret_cast<const Plan*>(plan);
        if (p.n_rows > 0 && !ml_part) { set_error("ml_part is NULL"); return F3S_ERR_INVALID_VALUE; }
        if (reinterpret_cast<uintptr_t>(ml_part) & 7) { set_error("ml_part must be 8-byte aligned"); return F3S_ERR_UNSUPPORTED; }
        if (max_ctas < 0) { set_error("max_ctas < 0"); return F3S_ERR_INVALID_VALUE; }
        if (kv_row_stride != 0 && (kv_row_stride < (int64_t)heads * d ||
                                   (kv_row_stride * (dtype == F3S_E4M3 ? 1 : 2)) % 16 != 0)) {
            set_error("kv_row_stride must be >= heads * d and a multiple of 16 bytes");
            return F3S_ERR_INVALID_VALUE;
        }
        if (p.n_rows == 0) return F3S_OK;
        AttnArgs a{&p, Q, K, V, O_part, scale, heads, d, dtype, true, stream};
        a.kv_ld = kv_row_stride;
        a.ml_out = ml_part;
        a.max_ctas = max_ctas;
        DeviceScope scope;
        F3S_CUDA_TRY(scope.enter(p.device));
        if (p.nnz == 0 || p.n_cols == 0) {  // no entries in this block: O = 0, (m, l) = (floor, 0)
            F3S_CUDA_TRY(cudaMemsetAsync(O_part, 0, sizeof(float) * (size_t)p.n_rows * heads * d, stream));
            return launch_fill_ml(ml_part, (int64_t)p.n_rows * heads, stream);
        }
        return launch_attention_sm100(a);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_merge(int32_t parts, const float* O_parts, const float* ml_parts, int64_t n_rows,
                               int32_t heads, int32_t d, float* O, cudaStream_t stream) {
    try {
        if (parts < 1 || parts > 32) { set_error("parts must be in [1, 32]"); return F3S_ERR_INVALID_VALUE; }
        if (n_rows < 0 || heads < 1 || (d != 64 && d != 128)) { set_error("bad sizes"); return F3S_ERR_INVALID_VALUE; }
        if (n_rows > 0 && (!O_parts || !ml_parts || !O)) { set_error("NULL pointer"); return F3S_ERR_INVALID_VALUE; }
        return launch_parts_merge(parts, O_parts, ml_parts, n_rows * heads, d, O, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_ex(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                            int32_t heads, int32_t d, f3s_dtype dtype, f3s_variant variant, cudaStream_t stream) {
    try {
        return run_attention(plan, Q, K, V, O, scale, heads, d, dtype, variant, stream);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_trace(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                               int32_t heads, int32_t d, f3s_dtype dtype, f3s_variant variant, uint64_t* trace,
                               int32_t trace_chunks, int32_t grid, cudaStream_t stream) {
    if (grid < 0) { set_error("bad trace arguments"); return F3S_ERR_INVALID_VALUE; }  // trace_chunks < 0: experiments
    try {
        return run_attention(plan, Q, K, V, O, scale, heads, d, dtype, variant, stream, trace, trace_chunks, grid);
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

static f3s_status attention_host_async_impl(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O,
                                            float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    f3s_status st = check_attention_args(plan, Q, K, V, O, scale, heads, d, dtype, false);
    if (st != F3S_OK) return st;
    Plan& p = *reinterpret_cast<Plan*>(plan);
    DeviceScope scope;
    F3S_CUDA_TRY(scope.enter(p.device));
    size_t qn = (size_t)p.n_rows * heads * d, kn = (size_t)p.n_cols * heads * d;
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t es = dtype == F3S_E4M3 ? 1 : 2;  // bytes per input element
    qn *= es;  // input sizes in bytes from here on; the output is fp32
    kn *= es;
    const size_t need = up(qn) + 2 * up(kn) + up(qn / es * 4);
    char* base = nullptr;
    {
        std::lock_guard<std::mutex> lock(p.staging_mu);
        Plan::Staging* sg = nullptr;
        for (auto& x : p.staging)
            if (x.stream == stream) sg = &x;
        if (!sg) {
            p.staging.push_back({stream, nullptr, 0});
            sg = &p.staging.back();
        }
        if (sg->bytes < need) {
            if (sg->ptr) {  // the stream's earlier calls may still use the old buffer
                F3S_CUDA_TRY(cudaStreamSynchronize(stream));
                cudaFree(sg->ptr);
            }
            sg->ptr = nullptr;
            sg->bytes = 0;
            F3S_CUDA_TRY(cudaMalloc(&sg->ptr, need));
            sg->bytes = need;
        }
        base = static_cast<char*>(sg->ptr);
    }
    void* dQ = base;
    void* dK = base + up(qn);
    void* dV = base + up(qn) + up(kn);
    float* dO = reinterpret_cast<float*>(base + up(qn) + 2 * up(kn));
    if (qn) F3S_CUDA_TRY(cudaMemcpyAsync(dQ, Q, qn, cudaMemcpyHostToDevice, stream));
    if (kn) {
        F3S_CUDA_TRY(cudaMemcpyAsync(dK, K, kn, cudaMemcpyHostToDevice, stream));
        F3S_CUDA_TRY(cudaMemcpyAsync(dV, V, kn, cudaMemcpyHostToDevice, stream));
    }
    st = run_attention(plan, dQ, dK, dV, dO, scale, heads, d, dtype, F3S_VARIANT_DEFAULT, stream);
    if (st != F3S_OK) return st;
    if (qn) F3S_CUDA_TRY(cudaMemcpyAsync(O, dO, qn / es * 4, cudaMemcpyDeviceToHost, stream));
    return F3S_OK;
}

f3s_status f3s_attention_host_async(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O,
                                    float scale, int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    try {
        return attention_host_async_impl(plan, Q, K, V, O, scale, heads, d, dtype, stream);
    } catch (const std::bad_alloc&) {
        return F3S_ERR_OUT_OF_MEMORY;
    } catch (...) {
        set_error("internal error");
        return F3S_ERR_INTERNAL;
    }
}

f3s_status f3s_attention_host(f3s_plan_t plan, const void* Q, const void* K, const void* V, float* O, float scale,
                              int32_t heads, int32_t d, f3s_dtype dtype, cudaStream_t stream) {
    f3s_status st = f3s_attention_host_async(plan, Q, K, V, O, scale, heads, d, dtype, stream);
    if (st != F3S_OK) return st;
    F3S_CUDA_TRY(cudaStreamSynchronize(stream));
    return F3S_OK;
}

// ---- partitioner (host) ---------------------------------------------------------------------
static f3s_status partition_impl(const int32_t* rp, int32_t n, const int32_t* cuts, int32_t n_cuts, int32_t parts,
                                 int32_t* bounds) {
    // candidate boundary c (row index) has prefix nnz rp[c] - rp[0]; bounds[p] is the
    // candidate whose prefix is closest to p*total/parts, never moving backwards.
    const int64_t total = (int64_t)rp[n] - rp[0];
    bounds[0] = 0;
    int32_t ci = 0;  // index into candidates
    auto cand = [&](int32_t i) -> int32_t { return cuts ? cuts[i] : std::min(16 * i, n); };
    const int32_t n_cand = cuts ? n_cuts : (n + 15) / 16 + 1;
    for (int32_t q = 1; q < parts; ++q) {
        const double target = (double)total * q / parts;
        while (ci + 1 < n_cand && (double)(rp[cand(ci + 1)] - rp[0]) < target) ++ci;
        int32_t best = ci;
        if (ci + 1 < n_cand) {
            const double lo = target - (double)(rp[cand(ci)] - rp[0]);
            const double hi = (double)(rp[cand(ci + 1)] - rp[0]) - target;
            if (hi < lo) best = ci + 1;
        }
        bounds[q] = std::max(bounds[q - 1], cand(best));
    }
    bounds[parts] = n;
    for (int32_t q = 1; q < parts; ++q) bounds[q] = std::min(bounds[q], n);
    return F3S_OK;
}

f3s_status f3s_partition_rows(const int32_t* row_ptr_host, int32_t n, int32_t parts, int32_t* bounds) {
    if (!row_ptr_host || !bounds || n < 0 || parts < 1) { set_error("bad partition arguments"); return F3S_ERR_INVALID_VALUE; }
    for (int32_t i = 0; i < n; ++i)
        if (row_ptr_host[i + 1] < row_ptr_host[i]) { set_error("row_ptr is not non-decreasing"); return F3S_ERR_INVALID_CSR; }
    return partition_impl(row_ptr_host, n, nullptr, 0, parts, bounds);
}

f3s_status f3s_partition_at(const int32_t* row_ptr_host, int32_t n, const int32_t* cuts, int32_t n_cuts,
                            int32_t parts, int32_t* bounds) {
    if (!row_ptr_host || !bounds || !cuts || n < 0 || parts < 1 || n_cuts < 1) {
        set_error("bad partition arguments");
        return F3S_ERR_INVALID_VALUE;
    }
    for (int32_t i = 0; i < n; ++i)
        if (row_ptr_host[i + 1] < row_ptr_host[i]) { set_error("row_ptr is not non-decreasing"); return F3S_ERR_INVALID_CSR; }
    for (int32_t i = 0; i < n_cuts; ++i)
        if (cuts[i] < 0 || cuts[i] > n || (i && cuts[i] < cuts[i - 1])) { set_error("cuts must be ascending in [0, n]"); return F3S_ERR_INVALID_VALUE; }
    return partition_impl(row_ptr_host, n, cuts, n_cuts, parts, bounds);
}

const char* f3s_status_string(f3s_status s) {
    switch (s) {
        case F3S_OK: return "F3S_OK";
        case F3S_ERR_INVALID_VALUE: return "F3S_ERR_INVALID_VALUE";
        case F3S_ERR_INVALID_CSR: return "F3S_ERR_INVALID_CSR";
        case F3S_ERR_UNSUPPORTED: return "F3S_ERR_UNSUPPORTED";
        case F3S_ERR_OUT_OF_MEMORY: return "F3S_ERR_OUT_OF_MEMORY";
        case F3S_ERR_CUDA: return "F3S_ERR_CUDA";
        case F3S_ERR_INTERNAL: return "F3S_ERR_INTERNAL";
    }
    return "F3S_ERR_UNKNOWN";
}

const char* f3s_last_error(void) { return g_last_error.c_str(); }

int64_t f3s_launch_count(void) { return g_launches.load(); }

}  // extern "C"
