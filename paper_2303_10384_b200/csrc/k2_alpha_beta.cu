// k2_alpha_beta.cu -- K2: forward (alpha) and backward (beta) scores over the T x (U+1) grid lattice as an
// anti-diagonal wavefront; plain RNN-T and the two W-Transducer variants.
//
// Recursions (DESIGN.md §"Path"; Eq.(1), §2.3, §3.2, §4.3):
//   alpha(0,0) = 0
//   alpha(t,u) = LSE( alpha(t-1,u) + X_b(t-1,u),  alpha(t,u-1) + X_y(t,u-1),
//                     [W, u=0, t>=1]  0                               (initial skips)
//                     [FF, (t,u)=(T-1,U)]  LSE_{t'<=T-2} alpha(t',U)  (final skips) )
//   log P      = LSE( alpha(T-1,U) + X_b(T-1,U),  [AI] LSE_{t'<=T-2} alpha(t',U) )
//   beta(T-1,U) = X_b(T-1,U)
//   beta(t,u)  = LSE( X_b(t,u) + beta(t+1,u) [t<T-1],  X_y(t,u) + beta(t,u+1) [u<U],
//                     [FF, u=U, t<T-1] beta(T-1,U),  [AI, u=U, t<T-1] 0,
//                     [W, (t,u)=(0,0)] LSE_{t'>=1} beta(t',0) )
//
// Cell (t,u) depends only on cells of diagonal t+u-1 (plus running skip accumulators owned by one
// thread), so diagonal d is one parallel step: thread u handles cell (d-u, u).  One CTA per
// (utterance, direction): grid = 2*B, the alpha and beta CTAs of an utterance run concurrently.
// Per step a thread needs one value from its neighbour (u-1 for alpha, u+1 for beta): a warp shuffle,
// plus a shared-memory hand-off across warp boundaries and one named barrier over the active warps
// (none at all when U_b+1 <= 32).  Its own (X_b, X_y) pair is one 8-byte load from the anti-diagonal-
// major lp array, software-prefetched kPrefetch diagonals ahead.  Accumulation is fp64; the LSE
// correction term runs in fp32 MUFU (reading R11).
#include "common.cuh"

namespace rnnt {
namespace {

constexpr int kPrefetch = 4;

__device__ __forceinline__ void named_barrier(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int kVariant>
__global__ void __launch_bounds__(kMaxUp1)
    k2_alpha_beta(const float2* __restrict__ lp, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int Tmax, int Umax,
                  int V, int blank, double* __restrict__ alpha, double* __restrict__ beta,
                  double* __restrict__ logp, float* __restrict__ losses) {
    constexpr bool kW = kVariant != kRnnt;
    __shared__ double xfer[2][kMaxUp1 / 32];

    const int b = blockIdx.x >> 1;
    const bool fwd = (blockIdx.x & 1) == 0;
    const int u = threadIdx.x;
    const int lane = u & 31, warp = u >> 5;
    const int T = T_b[b], U = U_b[b];

    // Validate the utterance (data-dependent errors -> NaN loss, zero grads in K3).
    const bool len_bad = (T < 1 || T > Tmax || U < 0 || U > Umax);
    int mybad = 0;
    if (!len_bad && u < U) {
        const int y = targets[static_cast<int64_t>(b) * Umax + u];
        mybad = (y < 0 || y >= V || y == blank);
    }
    if (__syncthreads_or(len_bad || mybad)) {
        if (fwd && u == 0) {
            logp[b] = __longlong_as_double(0x7ff8000000000000LL);
            losses[b] = __int_as_float(0x7fc00000);
        }
        return;
    }
    const int nact = ((U + 1 + 31) >> 5) << 5;  // threads in the warps that own cells
    if (u >= nact) return;
    const int nwarps = nact >> 5;

    const int Up1 = Umax + 1;
    const int Dmax = Tmax + Umax;
    const float2* lpu = lp + static_cast<int64_t>(b) * Dmax * Up1 + u;  // slot u of diagonal 0
    double* const tab = (fwd ? alpha : beta) + static_cast<int64_t>(b) * Tmax * Up1 + u;
    const int D = T + U;  // diagonals 0 .. T+U-1
    const unsigned full = 0xffffffffu;

    // Prefetch ring: pf[k] holds diagonal (d + k) of the traversal.
    float2 pf[kPrefetch];
    auto diag_of_step = [&](int i) { return fwd ? i : D - 1 - i; };
    auto load_lp = [&](int i) -> float2 {
        if (i >= D) return make_float2(0.f, 0.f);
        const int d = diag_of_step(i);
        const int t = d - u;
        if (t < 0 || t >= T || u > U) return make_float2(0.f, 0.f);
        return lpu[static_cast<int64_t>(d) * Up1];
    };
#pragma unroll
    for (int k = 0; k < kPrefetch; ++k) pf[k] = load_lp(k);

    if (fwd) {
        double self = -INFINITY;   // alpha(t-1,u) + X_b(t-1,u) for the cell this thread handles next
        double pub = -INFINITY;    // alpha(t,u) + X_y(t,u): what thread u+1 needs next step
        double skip = -INFINITY;   // LSE_{t' <= T-2} alpha(t', U)   (thread U only, W variants)
        for (int i0 = 0; i0 < D; i0 += kPrefetch) {
#pragma unroll
            for (int k = 0; k < kPrefetch; ++k) {
                const int d = i0 + k;
                if (d < D) {  // block-uniform
                    double nb = __shfl_up_sync(full, pub, 1);
                    if (lane == 0) nb = (warp > 0 && d > 0) ? xfer[(d - 1) & 1][warp - 1] : -INFINITY;
                    const float2 l = pf[k];
                    pf[k] = load_lp(d + kPrefetch);
                    const int t = d - u;
                    if (t >= 0 && t < T && u <= U) {
                        double cur;
                        if (d == 0) {
                            cur = 0.0;
                        } else {
                            cur = lse2(self, nb);
                            if (kW && u == 0) cur = lse2(cur, 0.0);  // initial skip (0,0)->(t,0)
                            if (kVariant == kForceFinal && u == U && t == T - 1) cur = lse2(cur, skip);
                        }
                        tab[static_cast<int64_t>(t) * Up1] = cur;
                        self = cur + static_cast<double>(l.x);
                        pub = (u < U) ? cur + static_cast<double>(l.y) : -INFINITY;
                        if (kW && u == U && t <= T - 2) skip = lse2(skip, cur);
                        if (u == U && t == T - 1) {
                            double lp_total = self;  // terminating blank (T-1,U) -> F
                            if (kVariant == kAllowIgnore) lp_total = lse2(lp_total, skip);
                            logp[b] = lp_total;
                            losses[b] = static_cast<float>(-lp_total);
                        }
                    } else {
                        pub = -INFINITY;
                    }
                    if (nwarps > 1) {
                        if (lane == 31) xfer[d & 1][warp] = pub;
                        named_barrier(nact);
                    }
                }
            }
        }
    } else {
        double self = -INFINITY;   // beta(t+1,u)
        double pub = -INFINITY;    // beta(t,u): what thread u-1 needs next step
        double fin = -INFINITY;    // beta(T-1,U)                   (thread U, force-final)
        double skip0 = -INFINITY;  // LSE_{t' >= 1} beta(t', 0)     (thread 0, W variants)
        for (int i0 = 0; i0 < D; i0 += kPrefetch) {
#pragma unroll
            for (int k = 0; k < kPrefetch; ++k) {
                const int i = i0 + k;
                if (i < D) {
                    const int d = D - 1 - i;
                    double nb = __shfl_down_sync(full, pub, 1);
                    if (lane == 31) nb = (warp + 1 < nwarps && i > 0) ? xfer[(i - 1) & 1][warp + 1] : -INFINITY;
                    const float2 l = pf[k];
                    pf[k] = load_lp(i + kPrefetch);
                    const int t = d - u;
                    if (t >= 0 && t < T && u <= U) {
                        double cur;
                        if (t == T - 1 && u == U) {
                            cur = static_cast<double>(l.x);  // terminating blank to F
                            fin = cur;
                        } else {
                            const double x1 = (t < T - 1) ? self + static_cast<double>(l.x) : -INFINITY;
                            const double x2 = (u < U) ? nb + static_cast<double>(l.y) : -INFINITY;
                            cur = lse2(x1, x2);
                            if (kVariant == kForceFinal && u == U) cur = lse2(cur, fin);
                            if (kVariant == kAllowIgnore && u == U) cur = lse2(cur, 0.0);
                            if (kW && t == 0 && u == 0) cur = lse2(cur, skip0);
                        }
                        if (kW && u == 0 && t >= 1) skip0 = lse2(skip0, cur);
                        tab[static_cast<int64_t>(t) * Up1] = cur;
                        self = cur;
                        pub = cur;
                    } else {
                        pub = -INFINITY;
                    }
                    if (nwarps > 1) {
                        if (lane == 0) xfer[i & 1][warp] = pub;
                        named_barrier(nact);
                    }
                }
            }
        }
    }
}

template <int kVariant>
void launch_variant(const Problem& p, const Workspace& w, cudaStream_t s, int threads) {
    k2_alpha_beta<kVariant><<<2 * p.B, threads, 0, s>>>(w.lp, p.targets, p.T_b, p.U_b, p.Tmax, p.Umax, p.V,
                                                        p.blank, w.alpha, w.beta, w.logp, p.losses);
}

}  // namespace

cudaError_t launch_k2_alpha_beta(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int threads = ((p.Umax + 1 + 31) / 32) * 32;
    switch (p.variant) {
        case kRnnt: launch_variant<kRnnt>(p, w, s, threads); break;
        case kForceFinal: launch_variant<kForceFinal>(p, w, s, threads); break;
        case kAllowIgnore: launch_variant<kAllowIgnore>(p, w, s, threads); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace rnnt
