// k4_viterbi.cu -- K4: Viterbi forced alignment over the grid lattice (max-plus wavefront + back-trace).
//
// PAPER.md §2.1: the lattice serves "model training and forced alignment tasks"; SURVEY §8(f) NEXT-2.
// Same arcs as the loss (K2; §2.3, W skips §3.2, §4.3), max instead of LSE:
//   delta(0,0) = 0,  delta(t,u) = max( delta(t-1,u) + X_b(t-1,u),  delta(t,u-1) + X_y(t,u-1),
//                                      [W, u=0, t>=1] 0 )
//   best = terminating blank / final skips as in K2 (force-final: max over (t',U) -> (T-1,U) then the
//          blank; allow-ignore: max of the terminating blank and the skips (t',U) -> F).
// Ties are broken in a fixed order (reading R21): blank arc, then label arc, then skip arc; among
// final skips the earliest source frame.  One CTA per utterance, thread u owns column u (one anti-diagonal
// per step: shuffle + one named barrier when the row spans several warps); operands are staged in registers
// a group of kPf steps ahead, as in K2.  Back-pointers (1 byte per cell)
// live in shared memory when Tmax x (Umax+1) fits (<= 200 KB), else in the workspace; delta is kept in the
// workspace (anti-diagonal major) for the final-skip reductions.  Thread 0 back-traces.
#include "common.cuh"

namespace rnnt {
namespace {

constexpr int kBpBlank = 0, kBpLabel = 1, kBpSkip = 2;
constexpr int kSmemBpLimit = 200 * 1024;

__device__ __forceinline__ void named_barrier_v(int nthreads) {
    asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
}

template <int kVariant, int kPf, int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads)
    k4_viterbi(const double2* __restrict__ lp, const int32_t* __restrict__ targets,
               const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int Tmax, int Umax, int V,
               int blank, double* __restrict__ delta_ws, uint8_t* __restrict__ bp_ws, int bp_in_smem,
               float* __restrict__ best_out, int32_t* __restrict__ frames, int32_t* __restrict__ span) {
    constexpr bool kW = kVariant != kRnnt;
    extern __shared__ uint8_t bp_smem[];
    __shared__ double xfer[2][32];
    __shared__ int s_end_t, s_skip;
    __shared__ double s_best;

    const int b = blockIdx.x;
    const int u = threadIdx.x;
    const int lane = u & 31, warp = u >> 5;
    const int T = T_b[b], U = U_b[b];
    const bool len_bad = (T < 1 || T > Tmax || U < 0 || U > Umax);
    int mybad = 0;
    if (!len_bad && u < U) {
        const int y = targets[static_cast<int64_t>(b) * Umax + u];
        mybad = (y < 0 || y >= V || y == blank);
    }
    for (int i = u; i < Umax; i += blockDim.x) frames[static_cast<int64_t>(b) * Umax + i] = -1;
    if (__syncthreads_or(len_bad || mybad)) {
        if (u == 0) {
            best_out[b] = __int_as_float(0x7fc00000);
            if (span) span[2 * b] = span[2 * b + 1] = -1;
        }
        return;
    }
    const int nwarps = (U + 1 + 31) >> 5;
    const int nthr = nwarps << 5;
    const int Up1 = Umax + 1, Dmax = Tmax + Umax, D = T + U;
    uint8_t* bp = bp_in_smem ? bp_smem : bp_ws + static_cast<int64_t>(b) * Tmax * Up1;  // [t][Up1]
    const double2* lpb = lp + static_cast<int64_t>(b) * Dmax * Up1;
    double* dlt = delta_ws + static_cast<int64_t>(b) * Dmax * Up1;

    if (warp < nwarps) {
        const unsigned full = 0xffffffffu;
        const int Teff = (u <= U) ? T : 0;
        // Operand staging as in K2: two register groups of kPf wavefront steps, group g+1 loading while
        // group g is consumed.  Loads past the last diagonal stay inside the padded lp array (kLpPad >= kPf).
        const double2* ld_ptr = lpb + u;
        double* st_ptr = dlt + u;
        double2 ga[kPf], gb[kPf];
        auto load_group = [&](double2 (&g)[kPf]) {
#pragma unroll
            for (int s = 0; s < kPf; ++s) {
                g[s] = ld_ptr[0];
                ld_ptr += Up1;
            }
        };
        load_group(ga);
        double self = (u == 0) ? 0.0 : -INFINITY;  // delta(t-1,u) + X_b(t-1,u); (0,0) = max(0, -inf) = 0
        double pub = -INFINITY;                     // delta(t,u) + X_y(t,u) for column u+1
        auto step_fn = [&](int d, const double2& x) {
            double left = __shfl_up_sync(full, pub, 1);
            if (nwarps > 1 && lane == 0) left = (warp > 0 && d > 0) ? xfer[(d - 1) & 1][warp - 1] : -INFINITY;
            const int t = d - u;
            const bool valid = static_cast<unsigned>(t) < static_cast<unsigned>(Teff);
            double nb = (u == 0) ? ((kW && t >= 1) ? 0.0 : -INFINITY) : left;  // initial skip (0,0)->(t,0)
            const bool take = nb > self;  // strict: ties keep the blank arc
            const double cur = take ? nb : self;
            if (valid) {
                *st_ptr = cur;
                bp[static_cast<int64_t>(t) * Up1 + u] =
                    static_cast<uint8_t>(take ? ((u == 0) ? kBpSkip : kBpLabel) : kBpBlank);
            }
            st_ptr += Up1;
            self = valid ? cur + x.x : -INFINITY;
            pub = valid ? cur + x.y : -INFINITY;
            if (nwarps > 1) {
                if (lane == 31) xfer[d & 1][warp] = pub;
                named_barrier_v(nthr);
            }
        };
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
        // Final arcs, by the warp owning column U.
        if (warp == (U >> 5)) {
            __syncwarp();
            double* const colU = dlt + U;  // + (t+U)*Up1 -> delta(t,U)
            double m = -INFINITY;
            int tm = -1;
            if (kW)
                for (int tp = lane; tp <= T - 2; tp += 32) {
                    const double v = __ldcg(colU + static_cast<int64_t>(tp + U) * Up1);
                    if (v > m) {
                        m = v;
                        tm = tp;
                    }
                }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {  // max, ties -> earliest frame
                const double m2 = __shfl_xor_sync(full, m, off);
                const int t2 = __shfl_xor_sync(full, tm, off);
                if (m2 > m || (m2 == m && t2 >= 0 && (tm < 0 || t2 < tm))) {
                    m = m2;
                    tm = t2;
                }
            }
            if (lane == (U & 31)) {
                const int64_t last = static_cast<int64_t>(T - 1 + U) * Up1;
                const double into = __ldcg(colU + last);
                const double xb = __ldcg(&lpb[last + U].x);
                int skip_from = -1;
                double total;
                if (kVariant == kForceFinal) {
                    double a = into;
                    if (m > a) {  // force-final skip (t*,U)->(T-1,U)
                        a = m;
                        skip_from = tm;
                    }
                    total = a + xb;
                } else if (kVariant == kAllowIgnore) {
                    total = into + xb;
                    if (m > total) {  // allow-ignore skip (t*,U)->F
                        total = m;
                        skip_from = tm;
                    }
                } else {
                    total = into + xb;
                }
                s_best = total;
                s_skip = skip_from;
                s_end_t = (skip_from >= 0) ? skip_from : T - 1;
            }
        }
    }
    __syncthreads();
    if (u != 0) return;
    const double total = s_best;
    // +inf only from +inf arc scores, i.e. a NaN in the utterance's logits (common.cuh kNanArc): reported as an
    // invalid utterance (NaN, frames and span -1)
    best_out[b] = total == INFINITY ? __int_as_float(0x7fc00000) : static_cast<float>(total);
    if (total == -INFINITY || total == INFINITY) {
        if (span) span[2 * b] = span[2 * b + 1] = -1;
        return;
    }
    // Back-trace from the cell the path leaves the grid through.
    int t = s_end_t, uu = U, start_t = 0;
    int32_t* fr = frames + static_cast<int64_t>(b) * Umax;
    while (t != 0 || uu != 0) {
        const int f = bp[static_cast<int64_t>(t) * Up1 + uu];
        if (f == kBpBlank) {
            t -= 1;
        } else if (f == kBpLabel) {
            fr[uu - 1] = t;
            uu -= 1;
        } else {
            start_t = t;  // entered column 0 through the initial skip (0,0)->(t,0)
            t = 0;
        }
    }
    if (span) {
        span[2 * b] = start_t;
        span[2 * b + 1] = s_end_t;
    }
}

template <int kVariant, int kPf, int kMaxThreads>
cudaError_t launch_t(const Problem& p, const Workspace& w, float* best, int32_t* frames, int32_t* span,
                     cudaStream_t s) {
    const int threads = ((p.Umax + 1 + 31) / 32) * 32;
    const int64_t bp_bytes = static_cast<int64_t>(p.Tmax) * (p.Umax + 1);
    const bool in_smem = bp_bytes <= kSmemBpLimit;
    const size_t smem = in_smem ? static_cast<size_t>(bp_bytes) : 0;
    auto kern = k4_viterbi<kVariant, kPf, kMaxThreads>;
    if (in_smem) {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBpLimit);
        if (e != cudaSuccess) return e;
    }
    kern<<<p.B, threads, smem, s>>>(w.lp, p.targets, p.T_b, p.U_b, p.Tmax, p.Umax, p.V, p.blank, w.alpha,
                                    reinterpret_cast<uint8_t*>(w.beta), in_smem ? 1 : 0, best, frames, span);
    return cudaGetLastError();
}

// Thread bound by Umax + 1 (one column per thread); the staging depth shrinks with the register budget.
template <int kVariant>
cudaError_t launch_v(const Problem& p, const Workspace& w, float* best, int32_t* frames, int32_t* span,
                     cudaStream_t s) {
    const int up1 = p.Umax + 1;
    if (up1 <= 32) return launch_t<kVariant, 16, 32>(p, w, best, frames, span, s);
    if (up1 <= 128) return launch_t<kVariant, 16, 128>(p, w, best, frames, span, s);
    if (up1 <= 256) return launch_t<kVariant, 16, 256>(p, w, best, frames, span, s);
    if (up1 <= 512) return launch_t<kVariant, 8, 512>(p, w, best, frames, span, s);
    return launch_t<kVariant, 4, 1024>(p, w, best, frames, span, s);
}

}  // namespace

cudaError_t launch_k4_viterbi(const Problem& p, const Workspace& w, float* best, int32_t* frames, int32_t* span,
                              cudaStream_t s) {
    switch (p.variant) {
        case kRnnt: return launch_v<kRnnt>(p, w, best, frames, span, s);
        case kForceFinal: return launch_v<kForceFinal>(p, w, best, frames, span, s);
        case kAllowIgnore: return launch_v<kAllowIgnore>(p, w, best, frames, span, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace rnnt
