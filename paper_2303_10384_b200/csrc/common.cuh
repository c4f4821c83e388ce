// common.cuh -- device helpers and the workspace layout shared by the three kernels (product code only;
// nothing here is shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rnnt_b200.h"

namespace rnnt {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kMaxUp1 = 4096;         // Umax + 1 limit of the one-CTA-per-utterance wavefront (K2: up to 8
                                      // columns per lane x 512 lanes)
constexpr int kMaxUp1Viterbi = 1024;  // K4 (forced alignment): one thread per column
constexpr int kRowWarpsPerBlock = 8;  // K1 / K3: one warp per (b,t,u) row, 8 rows per 256-thread block
constexpr int kLpPad = 16;            // diagonals of slack before/after the lp array (>= K2 staging group)

enum Variant : int { kRnnt = 0, kForceFinal = 1, kAllowIgnore = 2 };

// ---------------------------------------------------------------------------------------------------
// Workspace layout (all offsets 256-byte aligned).  Cell (b,t,u) of a padded [B][Tmax][Umax+1] grid.
//   lse    fp32   [B][Tmax][Up1]            log sum_v exp(z[b,t,u,v])                (K1 -> K3)
//   lp     double2 [B][Tmax+Umax][Up1]      (X[t,u,blank], X[t,u,y_u]) at diagonal d = t+u, slot u
//                                           (anti-diagonal major: one wavefront step reads one
//                                           contiguous run; kLpPad*Up1 entries of slack on both
//                                           ends so K2's prefetches need no bounds checks)  (K1 -> K2, K3)
//   alpha  fp64   [B][Tmax+Umax][Up1]      alpha(t,u) at diagonal t+u, slot u        (K2 -> K3)
//   beta   fp64   [B][Tmax+Umax][Up1]      beta(t,u)  at diagonal t+u, slot u        (K2 -> K3)
//   logp   fp64   [B]       log P_b from the forward pass (NaN = invalid utterance)  (K2 -> K3)
// ---------------------------------------------------------------------------------------------------
struct Workspace {
    float* lse;
    double2* lp;
    double* alpha;
    double* beta;
    double* logp;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t workspace_bytes(int64_t B, int64_t Tmax, int64_t Umax) {
    const int64_t Up1 = Umax + 1;
    size_t s = 0;
    s += align256(sizeof(float) * B * Tmax * Up1);
    s += align256(sizeof(double2) * (B * (Tmax + Umax) + 2 * kLpPad) * Up1);
    s += align256(sizeof(double) * B * (Tmax + Umax) * Up1);
    s += align256(sizeof(double) * B * (Tmax + Umax) * Up1);
    s += align256(sizeof(double) * B);
    return s;
}

inline Workspace carve(void* base, int64_t B, int64_t Tmax, int64_t Umax) {
    const int64_t Up1 = Umax + 1;
    char* p = static_cast<char*>(base);
    Workspace w;
    w.lse = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * B * Tmax * Up1);
    w.lp = reinterpret_cast<double2*>(p) + kLpPad * Up1;
    p += align256(sizeof(double2) * (B * (Tmax + Umax) + 2 * kLpPad) * Up1);
    w.alpha = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * B * (Tmax + Umax) * Up1);
    w.beta = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * B * (Tmax + Umax) * Up1);
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

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 / FMUL2 -- two lanes of work per issue slot).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 upk(f32x2 v) {
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// 2^x on both halves (two MUFU.EX2)
__device__ __forceinline__ f32x2 ex2x2(f32x2 a) {
    const float2 v = upk(a);
    return pk(ex2(v.x), ex2(v.y));
}
// three-input max (sm_100: FMNMX3)
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// log(e^a + e^b).  fp64 difference and max, fp32 MUFU correction.  -inf operands need no branch: if one
// side is -inf the correction is exactly 0; if both are, diff is NaN, fminf(NaN, 0) = 0 and the result is
// -inf + ln 2 = -inf.
// kNanArc: a NaN in a row's logits (R12) makes its lse NaN, but K2's LSE below can drop a NaN operand
// (its max is a compare and select), which would leave that utterance's loss finite.  The Populate step (K1 / K6)
// therefore hands K2 +inf arc scores for such a row: every LSE carries +inf through to log P = +inf, which K2
// reports as a NaN loss and the gradient passes treat as a non-finite log P (zero gradients), as for invalid
// targets.  (A NaN label score for an invalid label stays: K2 checks the labels itself.)

__device__ __forceinline__ double lse2f(double a, double b) {
    const double diff = a - b;
    const double m = (diff > 0.0) ? a : b;
    const float x = fminf(-fabsf(static_cast<float>(diff)) * kLog2e, 0.f);
    const float c = lg2(1.f + ex2(x)) * kLn2;
    return m + static_cast<double>(c);
}

// LSE over the 32 lanes of a warp; every lane ends with the same value (lse2f is symmetric).
__device__ __forceinline__ double warp_lse(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = lse2f(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// L2 eviction policy for the once-read joint tensor: evict-first, so the streamed logits do not push the
// (reused) workspace out of L2.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// ---------------------------------------------------------------------------------------------------
// Kernel launchers (defined in k1_lse_gather.cu, k2_alpha_beta.cu, k3_grad.cu).
// ---------------------------------------------------------------------------------------------------
struct Problem {
    const void* logits;  // fp32 / fp16 / bf16 per `dtype` (elem.cuh)
    const int32_t* targets;
    const int32_t* T_b;
    const int32_t* U_b;
    int B, Tmax, Umax, V, blank, variant;
    float* losses;
    void* grads;  // same storage type as logits, or nullptr
    const float* grad_scale;
    int dtype;
};

// K1; with w.lp == nullptr (and p.targets == nullptr) it writes the normalizer lse only (generic lattices).
cudaError_t launch_k1_lse_gather(const Problem& p, const Workspace& w, cudaStream_t s);
int lanes_per_row(int nvec);  // K1 / K3 row-group width for a row of nvec 128-bit vectors
cudaError_t launch_k2_alpha_beta(const Problem& p, const Workspace& w, cudaStream_t s);
cudaError_t launch_k3_grad(const Problem& p, const Workspace& w, cudaStream_t s);
cudaError_t launch_loss_sum(const float* losses, int B, double* out, cudaStream_t s);
cudaError_t launch_k4_viterbi(const Problem& p, const Workspace& w, float* best, int32_t* frames, int32_t* span,
                              cudaStream_t s);

// Internal streams / events of the chunk-overlapped launch schedules (rnnt_api.cu): per host thread and
// device, created once; nullptr if they cannot be created (callers then run sequentially).
constexpr int kMaxChunks = 4;
struct AuxPool {
    bool ready = false;
    cudaStream_t aux[kMaxChunks] = {};
    cudaEvent_t k1_done[kMaxChunks] = {}, k2_done[kMaxChunks] = {};
};
AuxPool* aux_pool();
// Number of utterance chunks for a call of B utterances and `elems` joint-tensor elements (1 = sequential).
int overlap_chunks(int64_t B, int64_t elems);

}  // namespace rnnt
