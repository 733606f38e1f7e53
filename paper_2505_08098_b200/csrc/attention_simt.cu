// attention_simt.cu — CUDA-core variant of the fused pass (F3S_VARIANT_SIMT).
//
// Same plan-driven dataflow as Alg.1 without tensor cores: one CTA per
// (row window, head) item taken in plan order (LPT), one warp per query row of the
// window.  The warp walks the window's compacted columns (sptd, Alg.1 l.7), keeps those whose
// mask has its row bit (bitmap, l.14), computes s = scale*q.k_j with a warp reduction (SDDMM,
// l.13), updates the running max/sum in fp32 (online softmax, l.16-18), rounds p to the input
// dtype (l.19, Tab.mixedp) and accumulates p*v_j in fp32 (SpMM, l.22); O = acc / l is
// written once (l.24), 0 for rows without entries (reading c4).
//
// It is the measured CUDA-core baseline for the tcgen05 kernel and an independent GPU
// cross-check in the tests; the default path is attention_sm100.cu.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.h"

namespace f3s {
namespace {

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ float round_to(float x);
template <> __device__ __forceinline__ float round_to<__half>(float x) { return __half2float(__float2half_rn(x)); }
template <> __device__ __forceinline__ float round_to<__nv_bfloat16>(float x) {
    return __bfloat162float(__float2bfloat16_rn(x));
}

template <int D, typename T>
__global__ void __launch_bounds__(512) k_attn_simt(const int32_t* __restrict__ rw_ptr, const int32_t* __restrict__ cols,
                                                   const uint16_t* __restrict__ masks, const int32_t* __restrict__ order,
                                                   int32_t n_rows, int H, const T* __restrict__ Q,
                                                   const T* __restrict__ K, const T* __restrict__ V,
                                                   float* __restrict__ O, float scale_log2) {
    constexpr int E = D / 32;  // features per lane
    const int item = blockIdx.x;
    const int k = order[item / H], h = item % H;
    const int i = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = 16 * (int64_t)k + i;
    if (row >= n_rows) return;
    const int64_t ld = (int64_t)H * D;
    float q[E], acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { q[e] = to_f(Q[row * ld + h * D + lane * E + e]); acc[e] = 0.f; }
    float m = -INFINITY, l = 0.f;
    const int32_t b = rw_ptr[k], e_ = rw_ptr[k + 1];
    for (int32_t p = b; p < e_; ++p) {
        if (!((masks[p] >> i) & 1)) continue;  // warp-uniform
        const int64_t j = cols[p];
        const T* kr = K + j * ld + h * D + lane * E;
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) s += q[e] * to_f(kr[e]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float x = s * scale_log2;
        const float m_new = fmaxf(m, x);
        const float alpha = exp2f(m - m_new);  // m = -inf on the first entry -> 0
        const float pe = exp2f(x - m_new);
        l = l * alpha + pe;                   // l from the unrounded p (reading c7)
        const float pr = round_to<T>(pe);     // E cast to the input dtype (Alg.1 l.19)
        const T* vr = V + j * ld + h * D + lane * E;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = acc[e] * alpha + pr * to_f(vr[e]);
        m = m_new;
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) O[row * ld + h * D + lane * E + e] = acc[e] * inv;
}

template <int D, typename T>
f3s_status launch(const AttnArgs& a) {
    const Plan& p = *a.plan;
    const int64_t items = (int64_t)p.num_rw * a.heads;
    if (items == 0) return F3S_OK;
    if (items > 0x7FFFFFFF) { set_error("too many work items"); return F3S_ERR_UNSUPPORTED; }
    k_attn_simt<D, T><<<(unsigned)items, 512, 0, a.stream>>>(
        p.rw_ptr, p.cols, p.masks, a.lpt ? p.rw_order : p.rw_natural, p.n_rows, a.heads,
        static_cast<const T*>(a.Q), static_cast<const T*>(a.K), static_cast<const T*>(a.V), a.O,
        a.scale * 1.4426950408889634f);
    count_launch();
    F3S_CUDA_TRY(cudaGetLastError());
    return F3S_OK;
}

}  // namespace

f3s_status launch_attention_simt(const AttnArgs& a) {
    if (a.dtype == F3S_FP16) return a.d == 64 ? launch<64, __half>(a) : launch<128, __half>(a);
    return a.d == 64 ? launch<64, __nv_bfloat16>(a) : launch<128, __nv_bfloat16>(a);
}

}  // namespace f3s
