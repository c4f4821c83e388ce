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

template <int kVariant, int kC, int kPf, int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads)
    k2_alpha_beta(const double2* __restrict__ lp, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int Tmax, int Umax,
                  int V, int blank, double* __restrict__ alpha, double* __restrict__ beta,
                  double* __restrict__ logp, float* __restrict__ losses) {
    constexpr bool kW = kVariant != kRnnt;
    constexpr bool kMultiWarp = kMaxThreads > 32;
    __shared__ double xfer[2][kMaxThreads / 32];

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
    const int nwarps = kMultiWarp ? (nact_lanes + 31) >> 5 : 1;  // single-warp instances: no smem, no barrier
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
        // One wavefront step d; x holds the step's (X_b, X_y) operands (staged a group ahead).
        auto fwd_step = [&](int d, const double2 (&x)[kC]) {
            double left = __shfl_up_sync(full, pub[kC - 1], 1);
            if (kMultiWarp && nwarps > 1 && lane == 0) left = (warp > 0 && d > 0) ? xfer[(d - 1) & 1][warp - 1] : -INFINITY;
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
                const double cur = lse2f(self[j], nb);
                if (valid) st_ptr[j] = cur;
                self[j] = valid ? cur + x[j].x : -INFINITY;
                pub[j] = valid ? cur + x[j].y : -INFINITY;  // X_y(t,U) = -inf: no label arc leaves row U
            }
            st_ptr += step;
            if (kMultiWarp && nwarps > 1) {
                if (lane == 31) xfer[d & 1][warp] = pub[kC - 1];
                named_barrier(nthr);
            }
        };
        run_groups(fwd_step);
        // The final cell (T-1,U) is the last wavefront step and nothing but log P depends on it, so the final
        // skip terms are applied afterwards by the warp owning column U: skip = LSE_{t'<=T-2} alpha(t',U)
        // from the stored column (a warp reduction, not a per-step accumulator on the critical path), then
        //   force-final:  alpha(T-1,U) <- LSE(alpha(T-1,U), skip),  log P = alpha(T-1,U) + X_b(T-1,U)
        //   allow-ignore: log P = LSE(alpha(T-1,U) + X_b(T-1,U), skip)
        const int ownerU = U / kC;
        if (warp == (ownerU >> 5)) {
            __syncwarp();
            double* const colU = alpha + static_cast<int64_t>(b) * Dmax * Up1 + U;  // + (t+U)*Up1 -> alpha(t,U)
            double skip = -INFINITY;
            if (kW) {
                for (int tp = lane; tp <= T - 2; tp += 32) skip = lse2f(skip, __ldcg(colU + static_cast<int64_t>(tp + U) * Up1));
                skip = warp_lse(skip);
            }
            if (lane == (ownerU & 31)) {
                const int64_t last = static_cast<int64_t>(T - 1 + U) * Up1;
                double a = __ldcg(colU + last);
                const double xb = __ldcg(&lp[static_cast<int64_t>(b) * Dmax * Up1 + last + U].x);
                if (kVariant == kForceFinal) {
                    a = lse2f(a, skip);
                    colU[last] = a;
                }
                double total = a + xb;  // terminating blank (T-1,U) -> F
                if (kVariant == kAllowIgnore) total = lse2f(total, skip);
                logp[b] = total;
                // log P = +inf only from +inf arc scores: a NaN in the utterance's logits (common.cuh kNanArc)
                losses[b] = total == INFINITY ? __int_as_float(0x7fc00000) : static_cast<float>(-total);
            }
        }
    } else {
        // self[j]: beta(t+1,u) (this column's previous cell); pub[j]: beta(t,u) for column u-1's next step.
        double fin = -INFINITY;    // beta(T-1,U)                  (lane owning column U, force-final)
        auto bwd_step = [&](int i, const double2 (&x)[kC]) {
            const int d = D - 1 - i;
            double right = __shfl_down_sync(full, pub[0], 1);
            if (kMultiWarp && nwarps > 1 && lane == 31)
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
                if (valid) st_ptr[j] = cur;
                if (kVariant == kForceFinal) fin = (valid && last) ? cur : fin;
                self[j] = valid ? cur : -INFINITY;
                pub[j] = self[j];
            }
            st_ptr += step;
            if (kMultiWarp && nwarps > 1) {
                if (lane == 0) xfer[i & 1][warp] = pub[0];
                named_barrier(nthr);
            }
        };
        run_groups(bwd_step);
        // Initial skips enter only beta(0,0) (the first cell, last step): warp 0 adds
        // LSE_{t'>=1} beta(t',0) from the stored column afterwards.  beta(0,0) = log P is the check value.
        if (kW && warp == 0) {
            __syncwarp();
            double* const col0 = beta + static_cast<int64_t>(b) * Dmax * Up1;  // + t*Up1 -> beta(t,0)
            double skip0 = -INFINITY;
            for (int tp = 1 + lane; tp <= T - 1; tp += 32) skip0 = lse2f(skip0, __ldcg(col0 + static_cast<int64_t>(tp) * Up1));
            skip0 = warp_lse(skip0);
            if (lane == 0) col0[0] = lse2f(__ldcg(col0), skip0);
        }
    }
}

template <int kVariant, int kC, int kPf, int kMaxThreads>
void launch_c(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int lanes = (p.Umax + 1 + kC - 1) / kC;
    const int threads = ((lanes + 31) / 32) * 32;
    k2_alpha_beta<kVariant, kC, kPf, kMaxThreads><<<2 * p.B, threads, 0, s>>>(
        w.lp, p.targets, p.T_b, p.U_b, p.Tmax, p.Umax, p.V, p.blank, w.alpha, w.beta, w.logp, p.losses);
}

// Shape of the wavefront CTA (columns per lane kC, staging group kPf, thread bound) by Umax + 1.
// Measured per step on B200 (T=500): one warp, 1 column per lane: 124 ns; one warp, 2 columns per lane:
// 160 ns; 2-4 warps, 1 column per lane (a named barrier per step): ~200 ns.  So a single warp while
// kC <= 2 covers the row, then one column per lane across warps; kPf shrinks as the per-thread register
// budget does (65536 / threads).  Beyond 1024 columns (long transcripts, U + 1 <= 4096): 512 lanes with 4 or 8
// columns each, kPf 2 or 1.  RNNT_K2_CELLS=1|2 forces kC where the table allows it (tuning knob).
template <int kVariant>
void launch_variant(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int up1 = p.Umax + 1;
    int force = 0;
    if (const char* e = getenv("RNNT_K2_CELLS")) force = atoi(e);
    if (up1 <= 32 && force != 2)
        launch_c<kVariant, 1, 16, 32>(p, w, s);
    else if (up1 <= 64 && force != 1)
        launch_c<kVariant, 2, 8, 32>(p, w, s);
    else if (up1 <= 128)
        launch_c<kVariant, 1, 16, 128>(p, w, s);
    else if (up1 <= 256 && force != 2)
        launch_c<kVariant, 1, 16, 256>(p, w, s);
    else if (up1 <= 512 && force != 2)
        launch_c<kVariant, 1, 8, 512>(p, w, s);
    else if (up1 <= 1024)
        launch_c<kVariant, 2, 4, 512>(p, w, s);
    else if (up1 <= 2048)  // long transcripts: more columns per lane, shallower operand staging (registers)
        launch_c<kVariant, 4, 2, 512>(p, w, s);
    else
        launch_c<kVariant, 8, 1, 512>(p, w, s);
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
