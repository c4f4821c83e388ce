// k5_lattice.cu -- the generic acyclic-lattice loss: any lattice whose arcs are bound to
// (t, u, v) of the joint logits or structural (weight 0) -- the Compose-/Grid-/W-Transducer graphs of
// PAPER.md §2.2-§3.2 and new topologies without new kernels.
//
//   L2 arc weights     w(a) = z[b,t,u,v] - lse[b,t,u]  (Populate, Eq.(3)), 0 for structural arcs
//   L3 forward/backward  level-synchronous: one CTA per (lattice, direction); the states of a level are
//                      independent (all arcs go to a higher level), so threads stride over the level, each
//                      state doing an fp64 LSE over its in- (alpha) or out-arcs (beta), one barrier per level.
//                      log P_b = beta(start).
//   L4 arc occupancies occ(a) = exp(alpha(src) + w(a) + beta(dst) - log P), summed per logits row
//                      (t,u) into S[b,t,u] (float atomics)
//   L5 row pass        grads[b,t,u,:] = softmax(z[b,t,u,:]) * S[b,t,u] for live rows, 0 elsewhere
//   L6 scatter         grads[b,t,u,v] -= occ(a) for every bound arc (float atomics)
// so d loss / d z = softmax * sum(occ) - occ, the chain rule through the log-softmax (reading R8).  fp32
// logits / grads.  Float atomics make the result order-dependent only where several arcs share a row (> 2)
// or a (t,u,v) (> 1); the grid lattices have at most 2 and 1.
#include "common.cuh"
#include "elem.cuh"
#include "rnnt_b200.h"

namespace rnnt {
namespace {

struct Lat {
    const int32_t *state_off, *lvl_off, *level_off, *in_off, *out_off, *out_arc;
    const int32_t *src, *dst, *t, *u, *v;
    const float* final_w;
};

__device__ __forceinline__ double lse2d(double a, double b) {
    const double m = fmax(a, b);
    if (m == -INFINITY) return m;
    return m + log1p(exp(fmin(a, b) - m));
}

// L2: one thread per arc of lattice blockIdx.y.
__global__ void __launch_bounds__(256) l2_arc_weights(const float* __restrict__ logits, const float* __restrict__ lse,
                                                      Lat L, int Tmax, int Umax, int V, float* __restrict__ w) {
    const int b = blockIdx.y;
    const int a0 = L.in_off[L.state_off[b]], a1 = L.in_off[L.state_off[b + 1]];
    const int64_t Up1 = Umax + 1;
    for (int a = a0 + static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); a < a1;
         a += static_cast<int>(gridDim.x * blockDim.x)) {
        const int v = L.v[a];
        float x = 0.f;
        if (v >= 0) {
            const int64_t row = (static_cast<int64_t>(b) * Tmax + L.t[a]) * Up1 + L.u[a];
            const float l = lse[row];
            x = (l == -INFINITY) ? -INFINITY : logits[row * V + v] - l;
        }
        w[a] = x;
    }
}

// L3: grid 2*B; even blocks forward, odd blocks backward.
__global__ void __launch_bounds__(256) l3_forward_backward(Lat L, const float* __restrict__ w, double* __restrict__ alpha,
                                                           double* __restrict__ beta, double* __restrict__ logp,
                                                           float* __restrict__ losses) {
    const int b = blockIdx.x >> 1;
    const bool fwd = (blockIdx.x & 1) == 0;
    const int l0 = L.lvl_off[b], l1 = L.lvl_off[b + 1];
    const int s_start = L.state_off[b];
    if (fwd) {
        for (int l = l0; l < l1; ++l) {
            for (int s = L.level_off[l] + threadIdx.x; s < L.level_off[l + 1]; s += blockDim.x) {
                double acc = (s == s_start) ? 0.0 : -INFINITY;
                for (int a = L.in_off[s]; a < L.in_off[s + 1]; ++a) acc = lse2d(acc, alpha[L.src[a]] + w[a]);
                alpha[s] = acc;
            }
            __syncthreads();
        }
    } else {
        for (int l = l1 - 1; l >= l0; --l) {
            for (int s = L.level_off[l] + threadIdx.x; s < L.level_off[l + 1]; s += blockDim.x) {
                double acc = static_cast<double>(L.final_w[s]);
                for (int k = L.out_off[s]; k < L.out_off[s + 1]; ++k) {
                    const int a = L.out_arc[k];
                    acc = lse2d(acc, w[a] + beta[L.dst[a]]);
                }
                beta[s] = acc;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            logp[b] = beta[s_start];
            losses[b] = static_cast<float>(-beta[s_start]);
        }
    }
}

__device__ __forceinline__ float arc_occ(const Lat& L, const float* w, const double* alpha, const double* beta,
                                         double lP, int a) {
    const double e = alpha[L.src[a]] + static_cast<double>(w[a]) + beta[L.dst[a]] - lP;
    return (e == -INFINITY || !isfinite(lP)) ? 0.f : static_cast<float>(exp(e));
}

// L4 (scatter=false): S[row] += occ;  L6 (scatter=true): grads[row, v] -= occ.
template <bool kScatter>
__global__ void __launch_bounds__(256) l46_occupancy(Lat L, const float* __restrict__ w, const double* __restrict__ alpha,
                                                     const double* __restrict__ beta, const double* __restrict__ logp,
                                                     int Tmax, int Umax, int V, float* __restrict__ rowS,
                                                     float* __restrict__ grads) {
    const int b = blockIdx.y;
    const int a0 = L.in_off[L.state_off[b]], a1 = L.in_off[L.state_off[b + 1]];
    const double lP = logp[b];
    const int64_t Up1 = Umax + 1;
    for (int a = a0 + static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); a < a1;
         a += static_cast<int>(gridDim.x * blockDim.x)) {
        const int v = L.v[a];
        if (v < 0) continue;
        const float o = arc_occ(L, w, alpha, beta, lP, a);
        if (o == 0.f) continue;
        const int64_t row = (static_cast<int64_t>(b) * Tmax + L.t[a]) * Up1 + L.u[a];
        if (kScatter)
            atomicAdd(grads + row * V + v, -o);
        else
            atomicAdd(rowS + row, o);
    }
}

// L5: warp per row; grads = softmax * S on live rows (t < T_b, u <= U_b, finite log P), zeros elsewhere.
__global__ void __launch_bounds__(256) l5_rows(const float* logits, const float* __restrict__ lse,
                                               const float* __restrict__ rowS, const int32_t* __restrict__ T_b,
                                               const int32_t* __restrict__ U_b, const double* __restrict__ logp,
                                               int Tmax, int Umax, int V, float* grads, bool vec4) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int Up1 = Umax + 1;
    const int r = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (r >= Tmax * Up1) return;
    const int t = r / Up1, u = r - t * Up1;
    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    const bool live = t < T_b[b] && u <= U_b[b] && isfinite(logp[b]);
    const float S = live ? rowS[row] : 0.f;
    const float l = live ? lse[row] : 0.f;
    const float* zr = logits + row * V;
    float* gr = grads + row * V;
    const bool on = live && S != 0.f && l != -INFINITY;
    const float ll = l * kLog2e;
    if (vec4) {  // 128-bit path: 8 loads per lane in flight
        const float4* z4 = reinterpret_cast<const float4*>(zr);
        float4* g4 = reinterpret_cast<float4*>(gr);
        const int nv = V >> 2;
        for (int base = 0; base < nv; base += 256) {
            float4 x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = base + j * 32 + lane;
                if (on && i < nv) x[j] = z4[i];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = base + j * 32 + lane;
                if (i < nv) {
                    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (on) {
                        g.x = ex2(fmaf(x[j].x, kLog2e, -ll)) * S;
                        g.y = ex2(fmaf(x[j].y, kLog2e, -ll)) * S;
                        g.z = ex2(fmaf(x[j].z, kLog2e, -ll)) * S;
                        g.w = ex2(fmaf(x[j].w, kLog2e, -ll)) * S;
                    }
                    g4[i] = g;
                }
            }
        }
        return;
    }
    for (int i = lane; i < V; i += 32) {
        const float g = on ? ex2((zr[i] - l) * kLog2e) * S : 0.f;
        gr[i] = g;
    }
}

}  // namespace

size_t lattice_workspace_bytes(int64_t B, int64_t Tmax, int64_t Umax, int64_t S, int64_t A) {
    const int64_t rows = B * Tmax * (Umax + 1);
    return align256(sizeof(float) * rows) * 2 + align256(sizeof(float) * A) + 2 * align256(sizeof(double) * S) +
           align256(sizeof(double) * B);
}

}  // namespace rnnt

using rnnt::Lat;

extern "C" size_t rnnt_lattice_workspace_bytes(int B, int Tmax, int Umax, int num_states, int num_arcs) {
    if (B < 0 || Tmax < 1 || Umax < 0 || num_states < 0 || num_arcs < 0) return 0;
    return rnnt::lattice_workspace_bytes(B, Tmax, Umax, num_states, num_arcs);
}

extern "C" rnnt_status rnnt_lattice_loss(const float* logits, const int32_t* logit_lens, const int32_t* target_lens,
                                         int B, int Tmax, int Umax, int V, const int32_t* state_off,
                                         const int32_t* lvl_off, const int32_t* level_off, const int32_t* in_off,
                                         const int32_t* out_off, const int32_t* out_arc, const int32_t* arc_src,
                                         const int32_t* arc_dst, const int32_t* arc_t, const int32_t* arc_u,
                                         const int32_t* arc_v, const float* final_w, int num_states, int num_arcs,
                                         float* losses, float* grads, void* workspace, size_t workspace_bytes,
                                         void* stream) {
    if (B < 0 || Tmax < 1 || Umax < 0 || V < 2 || num_states < 0 || num_arcs < 0) return RNNT_ERR_INVALID_ARG;
    if (B == 0) return RNNT_OK;
    if (!logits || !logit_lens || !target_lens || !state_off || !lvl_off || !level_off || !in_off || !out_off ||
        !final_w || !losses || !workspace || (num_arcs > 0 && (!out_arc || !arc_src || !arc_dst || !arc_t ||
                                                               !arc_u || !arc_v)))
        return RNNT_ERR_INVALID_ARG;
    if (workspace_bytes < rnnt::lattice_workspace_bytes(B, Tmax, Umax, num_states, num_arcs))
        return RNNT_ERR_WORKSPACE_TOO_SMALL;
    const int64_t rows = static_cast<int64_t>(B) * Tmax * (Umax + 1);
    char* p = static_cast<char*>(workspace);
    float* lse = reinterpret_cast<float*>(p);
    p += rnnt::align256(sizeof(float) * rows);
    float* rowS = reinterpret_cast<float*>(p);
    p += rnnt::align256(sizeof(float) * rows);
    float* w = reinterpret_cast<float*>(p);
    p += rnnt::align256(sizeof(float) * num_arcs);
    double* alpha = reinterpret_cast<double*>(p);
    p += rnnt::align256(sizeof(double) * num_states);
    double* beta = reinterpret_cast<double*>(p);
    p += rnnt::align256(sizeof(double) * num_states);
    double* logp = reinterpret_cast<double*>(p);

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Lat L{state_off, lvl_off, level_off, in_off, out_off, out_arc, arc_src, arc_dst, arc_t, arc_u, arc_v,
                final_w};
    // L1: the log-softmax normalizer of every live row (K1 without the grid gathers).
    rnnt::Problem pr{logits, nullptr, logit_lens, target_lens, B, Tmax, Umax, V, 0, rnnt::kRnnt, losses,
                     nullptr, nullptr, rnnt::kF32};
    rnnt::Workspace wk{lse, nullptr, nullptr, nullptr, nullptr};  // lp == nullptr: K1 writes lse only
    if (rnnt::launch_k1_lse_gather(pr, wk, s) != cudaSuccess) return RNNT_ERR_CUDA;
    const dim3 arc_grid(64, B);
    rnnt::l2_arc_weights<<<arc_grid, 256, 0, s>>>(logits, lse, L, Tmax, Umax, V, w);
    rnnt::l3_forward_backward<<<2 * B, 256, 0, s>>>(L, w, alpha, beta, logp, losses);
    if (grads) {
        if (cudaMemsetAsync(rowS, 0, sizeof(float) * rows, s) != cudaSuccess) return RNNT_ERR_CUDA;
        rnnt::l46_occupancy<false><<<arc_grid, 256, 0, s>>>(L, w, alpha, beta, logp, Tmax, Umax, V, rowS, grads);
        const int64_t bx = (static_cast<int64_t>(Tmax) * (Umax + 1) + 7) / 8;
        rnnt::l5_rows<<<dim3(static_cast<unsigned>(bx), B), 256, 0, s>>>(logits, lse, rowS, logit_lens, target_lens,
                                                                        logp, Tmax, Umax, V, grads,
                                                                        V % 4 == 0 && reinterpret_cast<uintptr_t>(logits) % 16 == 0 &&
                                                                            reinterpret_cast<uintptr_t>(grads) % 16 == 0);
        rnnt::l46_occupancy<true><<<arc_grid, 256, 0, s>>>(L, w, alpha, beta, logp, Tmax, Umax, V, rowS, grads);
    }
    return cudaGetLastError() == cudaSuccess ? RNNT_OK : RNNT_ERR_CUDA;
}
