// k2_alpha_beta.cu -- K2: forward (alpha) and backward (beta) scores over the T x (U+1) grid lattice as an
// anti-diagonal wavefront; plain RNN-T and the two W-Transducer variants.
//
// Recursions (Eq.(1), §2.3, §3.2, §4.3):
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
// Cell (t,u) depends only on cells of diagonal t+u-1 (plus skip accumulators owned by the lane holding
// column 0 / column U), so one anti-diagonal is one parallel step.  One CTA per (utterance, direction):
// grid = 2*B, the alpha and beta CTAs of an utterance run concurrently.  Lane l owns the kC consecutive
// columns u = l*kC .. l*kC+kC-1: per step its kC cells are independent LSE chains; the boundary column
// crosses lanes by one warp shuffle, and warps by a shared-memory slot + one named barrier per step
// (none when the utterance fits one warp).  The lp operands of a step are one contiguous run of the
// anti-diagonal-major fp64 lp array, staged through two register groups of kPf steps (group g+1 loads
// while group g computes; the array is padded by kLpPad diagonals on both ends, so loads need no bounds
// checks).  fp64 accumulation; the LSE
// correction log(1 + e^{-|a-b|}) is two MUFU ops in fp32 (reading R11).  alpha / beta are
// stored anti-diagonal major: [b][t+u][u].
#include <stdlib.h>

#include "common.cuh"

namespace rnnt {
namespace {

__device__ __forceinline__ void named_barrier(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// log(e^a + e^b).  fp64 difference and max, fp32 MUFU correction.  -inf operands need no branch: if one
// side is -inf the correction is exactly 0; if both are, diff is NaN, fminf(NaN, 0) = 0 and the result is
// -inf + ln 2 = -inf.
__device__ __forceinline__ double lse2f(double a, double b) {
    const double diff = a - b;
    const double m = (diff > 0.0) ? a : b;
    const float x = fminf(-fabsf(static_cast<float>(diff)) * kLog2e, 0.f);
    const float c = lg2(1.f + ex2(x)) * kLn2;
    return m + static_cast<double>(c);
}

template <int kVariant, int kC, int kPf>
__global__ void __launch_bounds__(128)
    k2_alpha_beta(const double2* __restrict__ lp, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int Tmax, int Umax,
                  int V, int blank, double* __restrict__ alpha, double* __restrict__ beta,
                  double* __restrict__ logp, float* __restrict__ losses) {
    constexpr bool kW = kVariant != kRnnt;
    __shared__ double xfer[2][4];

    const int b = blockIdx.x >> 1;
    const bool fwd = (blockIdx.x & 1) == 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int u0 = threadIdx.x * kC;  // first column of this lane
    const int T = T_b[b], U = U_b[b];

    // Validate the utterance (data-dependent errors -> NaN loss, zero grads in K3).
    const bool len_bad = (T < 1 || T > Tmax || U < 0 || U > Umax);
    int mybad = 0;
    if (!len_bad) {
#pragma unroll
        for (int j = 0; j < kC; ++j) {
            const int u = u0 + j;
            if (u < U) {
                const int y = targets[static_cast<int64_t>(b) * Umax + u];
                mybad |= (y < 0 || y >= V || y == blank);
            }
        }
    }
    if (__syncthreads_or(len_bad || mybad)) {
        if (fwd && threadIdx.x == 0) {
            logp[b] = __longlong_as_double(0x7ff8000000000000LL);
            losses[b] = __int_as_float(0x7fc00000);
        }
        return;
    }
    const int nact_lanes = (U + 1 + kC - 1) / kC;  // lanes owning at least one column
    const int nwarps = (nact_lanes + 31) >> 5;
    if (warp >= nwarps) return;
    const int nthr = nwarps << 5;

    const int Up1 = Umax + 1;
    const int Dmax = Tmax + Umax;
    const int D = T + U;  // diagonals 0 .. T+U-1
    const unsigned full = 0xffffffffu;
    const int64_t ubase = static_cast<int64_t>(b) * Dmax * Up1 + u0;
    // Per-cell validity: cell (d-u, u) exists iff 0 <= d-u < T and u <= U.
    int Teff[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) Teff[j] = (u0 + j <= U) ? T : 0;

    const int step = fwd ? Up1 : -Up1;        // pointer stride of one wavefront step
    const int d_first = fwd ? 0 : D - 1;
    const double2* ld_ptr = lp + ubase + static_cast<int64_t>(d_first) * Up1;  // padded: kPf steps of slack
    double* st_ptr = (fwd ? alpha : beta) + ubase + static_cast<int64_t>(d_first) * Up1;

    // Operand staging: two register groups of kPf steps each.  Group g+1 is loaded while group g is being
    // consumed, so every load has a whole group (kPf wavefront steps) to land.  Loads past the last
    // diagonal stay inside the padded lp array (kLpPad >= kPf diagonals of slack).
    double2 ga[kPf][kC], gb[kPf][kC];
    auto load_group = [&](double2 (&g)[kPf][kC]) {
#pragma unroll
        for (int s = 0; s < kPf; ++s) {
#pragma unroll
            for (int j = 0; j < kC; ++j) g[s][j] = ld_ptr[j];
            ld_ptr += step;
        }
    };
    load_group(ga);

    double self[kC], pub[kC];
#pragma unroll
    for (int j = 0; j < kC; ++j) self[j] = pub[j] = -INFINITY;

    // Drive steps 0 .. D-1 through the two staging groups (full groups run as straight-line code).
    auto run_groups = [&](auto&& step_fn) {
        for (int i0 = 0; i0 < D; i0 += 2 * kPf) {
            if (i0 + kPf < D) load_group(gb);
            if (i0 + kPf <= D) {
#pragma unroll
                for (int s = 0; s < kPf; ++s) step_fn(i0 + s, ga[s]);
            } else {
#pragma unroll
                for (int s = 0; s < kPf; ++s)
                    if (i0 + s < D) step_fn(i0 + s, ga[s]);
            }
            const int i1 = i0 + kPf;
            if (i1 >= D) break;
            if (i1 + kPf < D) load_group(ga);
            if (i1 + kPf <= D) {
#pragma unroll
                for (int s = 0; s < kPf; ++s) step_fn(i1 + s, gb[s]);
            } else {
#pragma unroll
                for (int s = 0; s < kPf; ++s)
                    if (i1 + s < D) step_fn(i1 + s, gb[s]);
            }
        }
    };

    if (fwd) {
        // self[j]: alpha(t-1,u) + X_b(t-1,u) for the next cell of column u0+j (column 0 starts at 0 so that
        // cell (0,0) = LSE(0, -inf) = 0 exactly).  pub[j]: alpha(t,u) + X_y(t,u) of the last computed cell.
        if (u0 == 0) self[0] = 0.0;
        double skip = -INFINITY;  // LSE_{t' <= T-2} alpha(t', U)   (lane owning column U, W variants)
        // One wavefront step d; x holds the step's (X_b, X_y) operands (staged a group ahead).
        auto fwd_step = [&](int d, const double2 (&x)[kC]) {
            double left = __shfl_up_sync(full, pub[kC - 1], 1);
            if (nwarps > 1 && lane == 0) left = (warp > 0 && d > 0) ? xfer[(d - 1) & 1][warp - 1] : -INFINITY;
            if (lane == 0 && warp == 0) left = -INFINITY;
#pragma unroll
            for (int j = kC - 1; j >= 0; --j) {  // high to low: pub[j-1] is still last step's
                const int u = u0 + j;
                const int t = d - u;
                const bool valid = static_cast<unsigned>(t) < static_cast<unsigned>(Teff[j]);
                double nb = (j == 0) ? left : pub[j - 1];
                // Column 0 has no left neighbour; under W its second incoming arc is the initial skip
                // (0,0)->(t,0) of weight 0, so one LSE per cell suffices on every column.
                if (kW && u == 0) nb = (t >= 1) ? 0.0 : -INFINITY;
                double cur = lse2f(self[j], nb);
                if (kVariant == kForceFinal && u == U && t == T - 1) cur = lse2f(cur, skip);  // once
                if (valid) st_ptr[j] = cur;
                self[j] = valid ? cur + x[j].x : -INFINITY;
                pub[j] = valid ? cur + x[j].y : -INFINITY;  // X_y(t,U) = -inf: no label arc leaves row U
                if (kW) {  // running LSE of alpha(t', U), t' <= T-2: computed by every lane, kept by column U
                    const double nskip = lse2f(skip, cur);
                    skip = (valid && u == U && t <= T - 2) ? nskip : skip;
                }
                if (valid && u == U && t == T - 1) {
                    double total = self[j];  // terminating blank (T-1,U) -> F
                    if (kVariant == kAllowIgnore) total = lse2f(total, skip);
                    logp[b] = total;
                    losses[b] = static_cast<float>(-total);
                }
            }
            st_ptr += step;
            if (nwarps > 1) {
                if (lane == 31) xfer[d & 1][warp] = pub[kC - 1];
                named_barrier(nthr);
            }
        };
        run_groups(fwd_step);
    } else {
        // self[j]: beta(t+1,u) (this column's previous cell); pub[j]: beta(t,u) for column u-1's next step.
        double fin = -INFINITY;    // beta(T-1,U)                  (lane owning column U, force-final)
        double skip0 = -INFINITY;  // LSE_{t' >= 1} beta(t', 0)    (lane 0, W variants)
        auto bwd_step = [&](int i, const double2 (&x)[kC]) {
            const int d = D - 1 - i;
            double right = __shfl_down_sync(full, pub[0], 1);
            if (nwarps > 1 && lane == 31)
                right = (warp + 1 < nwarps && i > 0) ? xfer[(i - 1) & 1][warp + 1] : -INFINITY;
#pragma unroll
            for (int j = 0; j < kC; ++j) {  // low to high: pub[j+1] is still last step's
                const int u = u0 + j;
                const int t = d - u;
                const bool valid = static_cast<unsigned>(t) < static_cast<unsigned>(Teff[j]);
                const bool last = (t == T - 1) && (u == U);  // terminating blank (T-1,U) -> F
                // Row U has no label arc; under W its second outgoing arc is the final skip (P:116 / P:167):
                // to (T-1,U) for force-final (beta(T-1,U)), to F for allow-ignore (0).
                double op2 = ((j == kC - 1) ? right : pub[j + 1]) + x[j].y;
                if (kVariant == kForceFinal && u == U) op2 = fin;
                if (kVariant == kAllowIgnore && u == U) op2 = 0.0;
                double cur = lse2f(self[j] + x[j].x, op2);
                cur = last ? x[j].x : cur;
                if (kW && t == 0 && u == 0) cur = lse2f(cur, skip0);  // initial skips, once
                if (valid) st_ptr[j] = cur;
                if (kVariant == kForceFinal) fin = (valid && last) ? cur : fin;
                if (kW) {  // running LSE of beta(t', 0), t' >= 1: computed by every lane, kept by column 0
                    const double nskip = lse2f(skip0, cur);
                    skip0 = (valid && u == 0 && t >= 1) ? nskip : skip0;
                }
                self[j] = valid ? cur : -INFINITY;
                pub[j] = self[j];
            }
            st_ptr += step;
            if (nwarps > 1) {
                if (lane == 0) xfer[i & 1][warp] = pub[0];
                named_barrier(nthr);
            }
        };
        run_groups(bwd_step);
    }
}

template <int kVariant, int kC, int kPf>
void launch_c(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int lanes = (p.Umax + 1 + kC - 1) / kC;
    const int threads = ((lanes + 31) / 32) * 32;
    k2_alpha_beta<kVariant, kC, kPf><<<2 * p.B, threads, 0, s>>>(w.lp, p.targets, p.T_b, p.U_b, p.Tmax, p.Umax,
                                                                 p.V, p.blank, w.alpha, w.beta, w.logp, p.losses);
}

// Columns per lane: the smallest kC that keeps the CTA within 4 warps (128 threads), unless the
// RNNT_K2_CELLS environment variable (1, 2, 4 or 8; a tuning knob) asks for more.
int cells_per_lane(int up1) {
    int c = (up1 <= 128) ? 1 : (up1 <= 256) ? 2 : (up1 <= 512) ? 4 : 8;
    if (const char* e = getenv("RNNT_K2_CELLS")) {
        const int want = atoi(e);
        if ((want == 1 || want == 2 || want == 4 || want == 8) && want > c) c = want;
    }
    return c;
}

template <int kVariant>
void launch_variant(const Problem& p, const Workspace& w, cudaStream_t s) {
    switch (cells_per_lane(p.Umax + 1)) {  // staging group = kPf steps, i.e. kPf..2*kPf steps of load slack
        case 1: launch_c<kVariant, 1, 16>(p, w, s); break;
        case 2: launch_c<kVariant, 2, 8>(p, w, s); break;
        case 4: launch_c<kVariant, 4, 4>(p, w, s); break;
        default: launch_c<kVariant, 8, 2>(p, w, s); break;
    }
}

}  // namespace

cudaError_t launch_k2_alpha_beta(const Problem& p, const Workspace& w, cudaStream_t s) {
    switch (p.variant) {
        case kRnnt: launch_variant<kRnnt>(p, w, s); break;
        case kForceFinal: launch_variant<kForceFinal>(p, w, s); break;
        case kAllowIgnore: launch_variant<kAllowIgnore>(p, w, s); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace rnnt
