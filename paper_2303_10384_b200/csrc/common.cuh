// common.cuh -- device helpers and the workspace layout shared by the three kernels (product code only;
// nothing here is shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rnnt_b200.h"

namespace rnnt {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kMaxUp1 = 1024;         // Umax + 1 limit of the one-CTA-per-utterance wavefront
constexpr int kRowWarpsPerBlock = 8;  // K1 / K3: one warp per (b,t,u) row, 8 rows per 256-thread block

enum Variant : int { kRnnt = 0, kForceFinal = 1, kAllowIgnore = 2 };

// ---------------------------------------------------------------------------------------------------
// Workspace layout (all offsets 256-byte aligned).  Cell (b,t,u) of a padded [B][Tmax][Umax+1] grid.
//   lse    fp32   [B][Tmax][Up1]            log sum_v exp(z[b,t,u,v])                (K1 -> K3)
//   lp     float2 [B][Tmax+Umax][Up1]       (X[t,u,blank], X[t,u,y_u]) at diagonal d = t+u, slot u
//                                           (anti-diagonal major: one wavefront step reads one
//                                           contiguous run)                          (K1 -> K2, K3)
//   alpha  fp64   [B][Tmax][Up1]                                                     (K2 -> K3)
//   beta   fp64   [B][Tmax][Up1]                                                     (K2 -> K3)
//   logp   fp64   [B]       log P_b from the forward pass (NaN = invalid utterance)  (K2 -> K3)
// ---------------------------------------------------------------------------------------------------
struct Workspace {
    float* lse;
    float2* lp;
    double* alpha;
    double* beta;
    double* logp;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t workspace_bytes(int64_t B, int64_t Tmax, int64_t Umax) {
    const int64_t Up1 = Umax + 1;
    size_t s = 0;
    s += align256(sizeof(float) * B * Tmax * Up1);
    s += align256(sizeof(float2) * B * (Tmax + Umax) * Up1);
    s += align256(sizeof(double) * B * Tmax * Up1);
    s += align256(sizeof(double) * B * Tmax * Up1);
    s += align256(sizeof(double) * B);
    return s;
}

inline Workspace carve(void* base, int64_t B, int64_t Tmax, int64_t Umax) {
    const int64_t Up1 = Umax + 1;
    char* p = static_cast<char*>(base);
    Workspace w;
    w.lse = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * B * Tmax * Up1);
    w.lp = reinterpret_cast<float2*>(p);
    p += align256(sizeof(float2) * B * (Tmax + Umax) * Up1);
    w.alpha = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * B * Tmax * Up1);
    w.beta = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * B * Tmax * Up1);
    w.logp = reinterpret_cast<double*>(p);
    return w;
}

// ---------------------------------------------------------------------------------------------------
// Fast transcendental helpers (MUFU).  ex2.approx.ftz: 2^x; lg2.approx.ftz: log2(x).
// ---------------------------------------------------------------------------------------------------
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Streaming loads/stores.  ld.global.nc.L1::no_allocate: read-only path, no L1 allocation (K1 only:
// logits are read-only there).  ld.global.cs / st.global.cs: evict-first streaming (K3, which may be in
// place, so it avoids the non-coherent path).
__device__ __forceinline__ float4 ld_stream_ro(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream_ro(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// log(e^a + e^b) with fp64 max/add and an fp32 log1p(exp(-|a-b|)) correction (reading R11:
// alpha/beta accumulate in fp64; the correction term is < ln 2 and needs only fp32 relative accuracy).
__device__ __forceinline__ double lse2(double a, double b) {
    const double m = fmax(a, b);
    if (m == -INFINITY) return -INFINITY;
    const float d = static_cast<float>(fmin(a, b) - m);  // <= 0, possibly -inf
    return m + static_cast<double>(log1pf(__expf(d)));
}

// ---------------------------------------------------------------------------------------------------
// Kernel launchers (defined in k1_lse_gather.cu, k2_alpha_beta.cu, k3_grad.cu).
// ---------------------------------------------------------------------------------------------------
struct Problem {
    const float* logits;
    const int32_t* targets;
    const int32_t* T_b;
    const int32_t* U_b;
    int B, Tmax, Umax, V, blank, variant;
    float* losses;
    float* grads;
    const float* grad_scale;
};

cudaError_t launch_k1_lse_gather(const Problem& p, const Workspace& w, cudaStream_t s);
cudaError_t launch_k2_alpha_beta(const Problem& p, const Workspace& w, cudaStream_t s);
cudaError_t launch_k3_grad(const Problem& p, const Workspace& w, cudaStream_t s);
cudaError_t launch_loss_sum(const float* losses, int B, double* out, cudaStream_t s);

}  // namespace rnnt
