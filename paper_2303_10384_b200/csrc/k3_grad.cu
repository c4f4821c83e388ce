// k3_grad.cu -- K3: arc occupancies and the fused logits-gradient, written in place or out of place.
//
// For a valid cell (t,u) of utterance b (S:257-270 arc posteriors; chain rule through X = log_softmax(z)):
//   occ_b = exp(alpha(t,u) + X_b(t,u) + beta(t+1,u) - logP)      t < T-1
//         = exp(alpha(T-1,U) + X_b(T-1,U) - logP)                 (t,u) = (T-1,U): terminating blank
//         = 0                                                     t = T-1, u < U (no blank arc leaves)
//   occ_y = exp(alpha(t,u) + X_y(t,u) + beta(t,u+1) - logP)       u < U, else 0
//   grad[v] = scale * ( softmax(z)[v] * (occ_b + occ_y) - [v == blank] occ_b - [v == y_u] occ_y )
// Skip arcs (W) carry no binding, so they contribute no gradient; their mass is why occ_b + occ_y need
// not equal exp(alpha + beta - logP).  Padded cells, invalid utterances (logP NaN) and no-path
// utterances (logP = -inf) get exact zeros, written without reading the logits.
//
// One warp per row; 128-bit loads and evict-first 128-bit stores; one ex2 per element.  In place is
// safe: every element is loaded by the thread that later stores its gradient, and rows never share data.
#include "common.cuh"

namespace rnnt {
namespace {

constexpr int kUnroll = 8;

template <bool kVec>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32)
    k3_grad(const float* logits, const int32_t* __restrict__ targets, const int32_t* __restrict__ T_b,
            const int32_t* __restrict__ U_b, int B, int Tmax, int Umax, int V, int blank,
            const float* __restrict__ grad_scale, const float* __restrict__ lse_in,
            const float2* __restrict__ lp_in, const double* __restrict__ alpha,
            const double* __restrict__ beta, const double* __restrict__ logp, float* grads) {
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5);
    const int Up1 = Umax + 1;
    const int64_t nrows = static_cast<int64_t>(B) * Tmax * Up1;
    if (row >= nrows) return;
    const int u = static_cast<int>(row % Up1);
    const int64_t bt = row / Up1;
    const int t = static_cast<int>(bt % Tmax);
    const int b = static_cast<int>(bt / Tmax);
    const int T = T_b[b], U = U_b[b];
    const double lP = logp[b];
    // Valid lengths are guaranteed whenever lP is finite (K2 writes NaN otherwise).
    const bool live = (t < T) && (u <= U) && isfinite(lP);

    float* grow = grads + row * static_cast<int64_t>(V);
    const float* zrow = logits + row * static_cast<int64_t>(V);

    if (!live) {
        if constexpr (kVec) {
            float4* g4 = reinterpret_cast<float4*>(grow);
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = lane; i < (V >> 2); i += 32) st_stream(g4 + i, zero);
        } else {
            for (int i = lane; i < V; i += 32) st_stream(grow + i, 0.f);
        }
        return;
    }

    // Per-row scalars: occupancies of the two scored arcs leaving (t,u).
    const int64_t cell = bt * Up1 + u;  // (b*Tmax + t)*Up1 + u
    const float lse = lse_in[cell];
    const float2 l = lp_in[(static_cast<int64_t>(b) * (Tmax + Umax) + (t + u)) * Up1 + u];
    const double a = alpha[cell];
    float occ_b = 0.f, occ_y = 0.f;
    if (t < T - 1)
        occ_b = __expf(static_cast<float>(a + static_cast<double>(l.x) + beta[cell + Up1] - lP));
    else if (u == U)
        occ_b = __expf(static_cast<float>(a + static_cast<double>(l.x) - lP));
    int yv = -1;
    if (u < U) {
        occ_y = __expf(static_cast<float>(a + static_cast<double>(l.y) + beta[cell + 1] - lP));
        yv = targets[static_cast<int64_t>(b) * Umax + u];
    }
    const float scale = grad_scale ? grad_scale[b] : 1.f;
    const float gam = (occ_b + occ_y) * scale;
    const float sb = occ_b * scale, sy = occ_y * scale;
    const float lsel = (lse == -INFINITY) ? INFINITY : lse * kLog2e;  // all -inf row -> p = 0

    if constexpr (kVec) {
        const float4* z4 = reinterpret_cast<const float4*>(zrow);
        float4* g4 = reinterpret_cast<float4*>(grow);
        const int nvec = V >> 2;
        for (int base = 0; base < nvec; base += 32 * kUnroll) {
            float4 x[kUnroll];
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) {
                const int i = base + j * 32 + lane;
                if (i < nvec) x[j] = ld_stream(z4 + i);
            }
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) {
                const int i = base + j * 32 + lane;
                if (i < nvec) {
                    const int v0 = i << 2;
                    float4 g;
                    g.x = ex2(fmaf(x[j].x, kLog2e, -lsel)) * gam - (v0 + 0 == blank ? sb : 0.f) - (v0 + 0 == yv ? sy : 0.f);
                    g.y = ex2(fmaf(x[j].y, kLog2e, -lsel)) * gam - (v0 + 1 == blank ? sb : 0.f) - (v0 + 1 == yv ? sy : 0.f);
                    g.z = ex2(fmaf(x[j].z, kLog2e, -lsel)) * gam - (v0 + 2 == blank ? sb : 0.f) - (v0 + 2 == yv ? sy : 0.f);
                    g.w = ex2(fmaf(x[j].w, kLog2e, -lsel)) * gam - (v0 + 3 == blank ? sb : 0.f) - (v0 + 3 == yv ? sy : 0.f);
                    st_stream(g4 + i, g);
                }
            }
        }
    } else {
        constexpr int kS = 4 * kUnroll;
        for (int base = 0; base < V; base += 32 * kS) {
            float x[kS];
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int i = base + j * 32 + lane;
                if (i < V) x[j] = ld_stream(zrow + i);
            }
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int i = base + j * 32 + lane;
                if (i < V) {
                    const float g = ex2(fmaf(x[j], kLog2e, -lsel)) * gam - (i == blank ? sb : 0.f) -
                                    (i == yv ? sy : 0.f);
                    st_stream(grow + i, g);
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch_k3_grad(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int64_t nrows = static_cast<int64_t>(p.B) * p.Tmax * (p.Umax + 1);
    const int64_t blocks = (nrows + kRowWarpsPerBlock - 1) / kRowWarpsPerBlock;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const bool vec = (p.V % 4 == 0) && (reinterpret_cast<uintptr_t>(p.logits) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(p.grads) % 16 == 0);
    if (vec)
        k3_grad<true><<<static_cast<unsigned>(blocks), kRowWarpsPerBlock * 32, 0, s>>>(
            p.logits, p.targets, p.T_b, p.U_b, p.B, p.Tmax, p.Umax, p.V, p.blank, p.grad_scale, w.lse,
            w.lp, w.alpha, w.beta, w.logp, p.grads);
    else
        k3_grad<false><<<static_cast<unsigned>(blocks), kRowWarpsPerBlock * 32, 0, s>>>(
            p.logits, p.targets, p.T_b, p.U_b, p.B, p.Tmax, p.Umax, p.V, p.blank, p.grad_scale, w.lse,
            w.lp, w.alpha, w.beta, w.logp, p.grads);
    return cudaGetLastError();
}

// Deterministic fp64 loss sum: one CTA, thread-strided partial sums then a fixed-shape tree.
__global__ void __launch_bounds__(256) k_loss_sum(const float* __restrict__ losses, int B, double* out) {
    __shared__ double part[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < B; i += 256) acc += static_cast<double>(losses[i]);
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) part[threadIdx.x] += part[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = part[0];
}

cudaError_t launch_loss_sum(const float* losses, int B, double* out, cudaStream_t s) {
    k_loss_sum<<<1, 256, 0, s>>>(losses, B, out);
    return cudaGetLastError();
}

}  // namespace rnnt
