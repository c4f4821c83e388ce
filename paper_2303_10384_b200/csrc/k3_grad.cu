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
// Wide rows: one warp per row (k3_grad_w); narrow rows (V/vector < 256): a group of 4..16 lanes per row
// (k3_grad_g), as K1.  128-bit loads and stores under an L2 evict-first policy; one ex2 per element;
// fp32 arithmetic, grads stored in the logits' storage type (fp32 / fp16 / bf16, round to nearest).  In
// place is safe: every element is loaded by the thread that later stores its gradient, and rows never
// share data.
#include "common.cuh"
#include "elem.cuh"

namespace rnnt {
namespace {

constexpr int kPerLane = 32;  // elements per lane per chunk

template <typename Z, bool kVec, typename VecT = uint4>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32)
    k3_grad_w(const Z* logits, const int32_t* __restrict__ targets, const int32_t* __restrict__ T_b,
            const int32_t* __restrict__ U_b, int b0, int Tmax, int Umax, int V, int blank,
            const float* __restrict__ grad_scale, const float* __restrict__ lse_in,
            const double2* __restrict__ lp_in, const double* __restrict__ alpha,
            const double* __restrict__ beta, const double* __restrict__ logp, Z* grads) {
    const int lane = threadIdx.x & 31;
    const int b = b0 + static_cast<int>(blockIdx.y);
    const int Up1 = Umax + 1;
    const int r = static_cast<int>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5);  // row in utterance
    if (r >= Tmax * Up1) return;
    const int t = r / Up1;
    const int u = r - t * Up1;
    const int T = T_b[b], U = U_b[b];
    const double lP = logp[b];
    // Valid lengths are guaranteed whenever lP is finite (K2 writes NaN otherwise).
    const bool live = (t < T) && (u <= U) && isfinite(lP);

    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    Z* grow = grads + row * static_cast<int64_t>(V);
    const Z* zrow = logits + row * static_cast<int64_t>(V);
    constexpr int E = static_cast<int>(sizeof(VecT) / sizeof(Z));

    if (!live) {
        if constexpr (kVec) {
            const uint64_t pol = l2_evict_first();
            VecT* g4 = reinterpret_cast<VecT*>(grow);
            for (int i = lane; i < V / E; i += 32) stv(g4 + i, zero_vec<VecT>(), pol);
        } else {
            for (int i = lane; i < V; i += 32) grow[i] = Elem<Z>::from_f32(0.f);
        }
        return;
    }

    constexpr int kU = kPerLane / E;
    const uint64_t pol = l2_evict_first();
    const VecT* z4 = reinterpret_cast<const VecT*>(zrow);
    const int nvec = V / E;
    VecT raw[kU];
    if constexpr (kVec) {  // issue the row's first chunk before the per-row scalars: both latencies overlap
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int i = j * 32 + lane;
            if (i < nvec) raw[j] = ldv(z4 + i, pol);
        }
    }

    // Per-row scalars: occupancies of the two scored arcs leaving (t,u).
    const int64_t dcell = (static_cast<int64_t>(b) * (Tmax + Umax) + (t + u)) * Up1 + u;  // diagonal t+u, slot u
    const float lse = lse_in[row];
    const double2 l = lp_in[dcell];
    const double a = alpha[dcell];
    float occ_b = 0.f, occ_y = 0.f;
    if (t < T - 1)  // beta(t+1,u): diagonal t+u+1, slot u
        occ_b = __expf(static_cast<float>(a + l.x + beta[dcell + Up1] - lP));
    else if (u == U)
        occ_b = __expf(static_cast<float>(a + l.x - lP));
    int yv = -1;
    if (u < U) {    // beta(t,u+1): diagonal t+u+1, slot u+1
        occ_y = __expf(static_cast<float>(a + l.y + beta[dcell + Up1 + 1] - lP));
        yv = targets[static_cast<int64_t>(b) * Umax + u];
    }
    const float scale = grad_scale ? grad_scale[b] : 1.f;
    const float gam = (occ_b + occ_y) * scale;
    const float sb = occ_b * scale, sy = occ_y * scale;
    const float lsel = (lse == -INFINITY) ? INFINITY : lse * kLog2e;  // all -inf row -> p = 0

    if constexpr (kVec) {
        VecT* g4 = reinterpret_cast<VecT*>(grow);
        const int bq = blank / E, yq = (yv < 0) ? -1 : (yv / E);
        const int bk = blank % E, yk = (yv < 0) ? 0 : (yv % E);
        const f32x2 l2e = pk(kLog2e, kLog2e), nl = pk(-lsel, -lsel), g2 = pk(gam, gam);
        for (int base = 0; base < nvec; base += 32 * kU) {
            if (base > 0) {
#pragma unroll
                for (int j = 0; j < kU; ++j) {
                    const int i = base + j * 32 + lane;
                    if (i < nvec) raw[j] = ldv(z4 + i, pol);
                }
            }
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                const int i = base + j * 32 + lane;
                if (i < nvec) {
                    float x[E], g[E];
                    Elem<Z>::unpack(raw[j], x);
#pragma unroll
                    for (int e = 0; e < E; e += 2) {
                        const float2 p = upk(fmul2(ex2x2(ffma2(pk(x[e], x[e + 1]), l2e, nl)), g2));
                        g[e] = p.x;
                        g[e + 1] = p.y;
                    }
                    if (i == bq) {  // the arcs' own logits: subtract their occupancies (owner lane only)
#pragma unroll
                        for (int e = 0; e < E; ++e) g[e] -= (e == bk) ? sb : 0.f;
                    }
                    if (i == yq) {
#pragma unroll
                        for (int e = 0; e < E; ++e) g[e] -= (e == yk) ? sy : 0.f;
                    }
                    stv(g4 + i, Elem<Z>::pack(g), pol);
                }
            }
        }
    } else {
        for (int base = 0; base < V; base += 32 * kPerLane) {
            float x[kPerLane];
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = base + j * 32 + lane;
                if (i < V) x[j] = Elem<Z>::to_f32(zrow[i]);
            }
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = base + j * 32 + lane;
                if (i < V) {
                    const float g = ex2(fmaf(x[j], kLog2e, -lsel)) * gam - (i == blank ? sb : 0.f) -
                                    (i == yv ? sy : 0.f);
                    grow[i] = Elem<Z>::from_f32(g);
                }
            }
        }
    }
}


constexpr int kVecPerLane = 8;  // 128-bit vectors per lane per chunk

// G lanes per (b,t,u) row (G = 4..32, see lanes_per_row): a warp keeps 8 x 128-bit loads per lane in
// flight whatever V and the storage type, exactly as K1.
template <typename Z, int G, typename VecT = uint4>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32)
    k3_grad_g(const Z* logits, const int32_t* __restrict__ targets, const int32_t* __restrict__ T_b,
            const int32_t* __restrict__ U_b, int b0, int Tmax, int Umax, int V, int blank,
            const float* __restrict__ grad_scale, const float* __restrict__ lse_in,
            const double2* __restrict__ lp_in, const double* __restrict__ alpha,
            const double* __restrict__ beta, const double* __restrict__ logp, Z* grads) {
    constexpr int E = static_cast<int>(sizeof(VecT) / sizeof(Z)), kU = kVecPerLane, kRowsPerWarp = 32 / G;
    const int lane = threadIdx.x & 31;
    const int sl = lane & (G - 1);
    const int b = b0 + static_cast<int>(blockIdx.y);
    const int Up1 = Umax + 1;
    const int r = (static_cast<int>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5)) * kRowsPerWarp + lane / G;
    if (r >= Tmax * Up1) return;  // no shuffles below: groups are independent
    const int t = r / Up1;
    const int u = r - t * Up1;
    const int T = T_b[b], U = U_b[b];
    const double lP = logp[b];
    // Valid lengths are guaranteed whenever lP is finite (K2 writes NaN otherwise).
    const bool live = (t < T) && (u <= U) && isfinite(lP);

    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    const uint64_t pol = l2_evict_first();
    VecT* g4 = reinterpret_cast<VecT*>(grads + row * static_cast<int64_t>(V));
    const VecT* z4 = reinterpret_cast<const VecT*>(logits + row * static_cast<int64_t>(V));
    const int nvec = V / E;

    if (!live) {  // padding / invalid / no-path: exact zeros, the logits are never read
        for (int i = sl; i < nvec; i += G) stv(g4 + i, zero_vec<VecT>(), pol);
        return;
    }

    VecT raw[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {  // the row's first chunk, issued before the per-row scalars
        const int i = j * G + sl;
        if (i < nvec) raw[j] = ldv(z4 + i, pol);
    }

    // Per-row scalars: occupancies of the two scored arcs leaving (t,u).
    const int64_t dcell = (static_cast<int64_t>(b) * (Tmax + Umax) + (t + u)) * Up1 + u;  // diagonal t+u, slot u
    const float lse = lse_in[row];
    const double2 l = lp_in[dcell];
    const double a = alpha[dcell];
    float occ_b = 0.f, occ_y = 0.f;
    if (t < T - 1)  // beta(t+1,u): diagonal t+u+1, slot u
        occ_b = __expf(static_cast<float>(a + l.x + beta[dcell + Up1] - lP));
    else if (u == U)
        occ_b = __expf(static_cast<float>(a + l.x - lP));
    int yv = -1;
    if (u < U) {    // beta(t,u+1): diagonal t+u+1, slot u+1
        occ_y = __expf(static_cast<float>(a + l.y + beta[dcell + Up1 + 1] - lP));
        yv = targets[static_cast<int64_t>(b) * Umax + u];
    }
    const float scale = grad_scale ? grad_scale[b] : 1.f;
    const float gam = (occ_b + occ_y) * scale;
    const float sb = occ_b * scale, sy = occ_y * scale;
    const float lsel = (lse == -INFINITY) ? INFINITY : lse * kLog2e;  // all -inf row -> p = 0

    const int bq = blank / E, yq = (yv < 0) ? -1 : (yv / E);
    const int bk = blank % E, yk = (yv < 0) ? 0 : (yv % E);
    const f32x2 l2e = pk(kLog2e, kLog2e), nl = pk(-lsel, -lsel), g2 = pk(gam, gam);
    for (int base = 0; base < nvec; base += G * kU) {
        if (base > 0) {
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                const int i = base + j * G + sl;
                if (i < nvec) raw[j] = ldv(z4 + i, pol);
            }
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int i = base + j * G + sl;
            if (i < nvec) {
                float x[E], g[E];
                Elem<Z>::unpack(raw[j], x);
#pragma unroll
                for (int e = 0; e < E; e += 2) {
                    const float2 q = upk(fmul2(ex2x2(ffma2(pk(x[e], x[e + 1]), l2e, nl)), g2));
                    g[e] = q.x;
                    g[e + 1] = q.y;
                }
                if (i == bq) {  // the arcs' own logits: subtract their occupancies (owner lane only)
#pragma unroll
                    for (int e = 0; e < E; ++e) g[e] -= (e == bk) ? sb : 0.f;
                }
                if (i == yq) {
#pragma unroll
                    for (int e = 0; e < E; ++e) g[e] -= (e == yk) ? sy : 0.f;
                }
                stv(g4 + i, Elem<Z>::pack(g), pol);
            }
        }
    }
}

template <typename Z, int G, typename VecT = uint4>
void launch_g(const Problem& p, const Workspace& w, cudaStream_t s, const Z* z, Z* g, int64_t rows_per_utt) {
    constexpr int kRowsPerBlock = kRowWarpsPerBlock * (32 / G);
    const int64_t bx = (rows_per_utt + kRowsPerBlock - 1) / kRowsPerBlock;
    for (int b0 = 0; b0 < p.B; b0 += 65535) {
        const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(min(65535, p.B - b0)));
        k3_grad_g<Z, G, VecT><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax,
                                                                 p.V, p.blank, p.grad_scale, w.lse, w.lp, w.alpha,
                                                                 w.beta, w.logp, g);
    }
}

template <typename Z>
cudaError_t launch_t(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int64_t rows_per_utt = static_cast<int64_t>(p.Tmax) * (p.Umax + 1);
    if (rows_per_utt > 0x7fffffffLL / 2) return cudaErrorInvalidConfiguration;
    const Z* z = static_cast<const Z*>(p.logits);
    Z* g = static_cast<Z*>(p.grads);
    constexpr int E = Elem<Z>::kPerVec;
    const bool vec = (p.V % E == 0) && (reinterpret_cast<uintptr_t>(z) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(g) % 16 == 0);
    const int lanes = vec ? lanes_per_row(p.V / E) : 32;
    if (lanes < 32) {  // narrow rows: grouped kernel
        switch (lanes) {
            case 4: launch_g<Z, 4>(p, w, s, z, g, rows_per_utt); break;
            case 8: launch_g<Z, 8>(p, w, s, z, g, rows_per_utt); break;
            default: launch_g<Z, 16>(p, w, s, z, g, rows_per_utt); break;
        }
        return cudaGetLastError();
    }
    // 64-bit vectors: 16-bit rows with V % 8 == 4 (e.g. V = 500), fp32 rows with V % 4 == 2
    const bool vec8 = !vec && (p.V % (8 / sizeof(Z)) == 0) && (reinterpret_cast<uintptr_t>(z) % 8 == 0) &&
                      (reinterpret_cast<uintptr_t>(g) % 8 == 0);
    const int lanes8 = vec8 ? lanes_per_row(static_cast<int>(p.V / (8 / sizeof(Z)))) : 32;
    if (vec8 && lanes8 < 32) {  // narrow 64-bit rows: grouped kernel, 8 x 64-bit loads per lane
        switch (lanes8) {
            case 4: launch_g<Z, 4, uint2>(p, w, s, z, g, rows_per_utt); break;
            case 8: launch_g<Z, 8, uint2>(p, w, s, z, g, rows_per_utt); break;
            default: launch_g<Z, 16, uint2>(p, w, s, z, g, rows_per_utt); break;
        }
        return cudaGetLastError();
    }
    const int64_t bx = (rows_per_utt + kRowWarpsPerBlock - 1) / kRowWarpsPerBlock;
    for (int b0 = 0; b0 < p.B; b0 += 65535) {
        const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(min(65535, p.B - b0)));
        if (vec8) {
                k3_grad_w<Z, true, uint2><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                    z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, p.grad_scale, w.lse, w.lp, w.alpha,
                    w.beta, w.logp, g);
        } else if (vec)
            k3_grad_w<Z, true><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, p.grad_scale, w.lse, w.lp, w.alpha,
                w.beta, w.logp, g);
        else
            k3_grad_w<Z, false><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, p.grad_scale, w.lse, w.lp, w.alpha,
                w.beta, w.logp, g);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_k3_grad(const Problem& p, const Workspace& w, cudaStream_t s) {
    switch (p.dtype) {
        case kF32: return launch_t<float>(p, w, s);
        case kF16: return launch_t<__half>(p, w, s);
        case kBF16: return launch_t<__nv_bfloat16>(p, w, s);
    }
    return cudaErrorInvalidValue;
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
