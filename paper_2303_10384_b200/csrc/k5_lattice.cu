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
                                                      Lat L, int Tmax, int Umax, int V, float* __restrict__ w, int b0) {
    const int b = b0 + blockIdx.y;
    const int a0 = L.in_off[L.state_off[b]], a1 = L.in_off[L.state_off[b + 1]];
    const int64_t Up1 = Umax + 1;
    for (int a = a0 + static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); a < a1;
         a += static_cast<int>(gridDim.x * blockDim.x)) {
        const int v = L.v[a];
        float x = 0.f;
        if (v >= 0) {
            const int64_t row = (static_cast<int64_t>(b) * Tmax + L.t[a]) * Up1 + L.u[a];
            const float l = lse[row];
            // a NaN in the row (lse NaN): +inf, as the grid path's Populate (common.cuh kNanArc), so that log P
            // becomes +inf and the loss NaN instead of a NaN operand being dropped by an LSE
            x = (l == -INFINITY) ? -INFINITY : (l != l) ? INFINITY : logits[row * V + v] - l;
        }
        w[a] = x;
    }
}

// Per-state record of one direction (built by l3_pack, read by l3_forward_backward): the first two arcs'
// neighbour state (src for alpha, dst for beta) and weight, the state's arc range (for the rest) and its
// initial value (alpha: 0 at the start state; beta: the log final weight).  One 32-byte load per state and
// level, one hop from the level table, so it can be fetched kPf levels ahead.  Every field is read: a dead
// word of an in-flight 128-bit load lets the register allocator reuse its register, and the reuse then
// waits for the load (a write-after-write stall of a full memory latency per level).
struct __align__(16) StateRec {
    int n0, n1;
    float w0, w1;
    int k0, kend;  // arc range [k0, kend)
    float init;
    int deg;       // kend - k0
};

// L3 pack: one thread per state of lattice b0 + blockIdx.y.
__global__ void __launch_bounds__(256) l3_pack(Lat L, const float* __restrict__ w, StateRec* __restrict__ rec_f,
                                               StateRec* __restrict__ rec_b, int b0) {
    const int b = b0 + blockIdx.y;
    const int s0 = L.state_off[b], s1 = L.state_off[b + 1];
    for (int s = s0 + static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x); s < s1;
         s += static_cast<int>(gridDim.x * blockDim.x)) {
        StateRec f{}, r{};
        f.k0 = L.in_off[s];
        f.kend = L.in_off[s + 1];
        f.deg = f.kend - f.k0;
        f.n0 = f.deg > 0 ? L.src[f.k0] : s;
        f.w0 = f.deg > 0 ? w[f.k0] : -INFINITY;
        f.n1 = f.deg > 1 ? L.src[f.k0 + 1] : s;
        f.w1 = f.deg > 1 ? w[f.k0 + 1] : -INFINITY;
        f.init = (s == s0) ? 0.f : -INFINITY;
        r.k0 = L.out_off[s];
        r.kend = L.out_off[s + 1];
        r.deg = r.kend - r.k0;
        const int a0 = r.deg > 0 ? L.out_arc[r.k0] : -1, a1 = r.deg > 1 ? L.out_arc[r.k0 + 1] : -1;
        r.n0 = a0 >= 0 ? L.dst[a0] : s;
        r.w0 = a0 >= 0 ? w[a0] : -INFINITY;
        r.n1 = a1 >= 0 ? L.dst[a1] : s;
        r.w1 = a1 >= 0 ? w[a1] : -INFINITY;
        r.init = L.final_w[s];
        rec_f[s] = f;
        rec_b[s] = r;
    }
}

constexpr int kL3Threads = 512;
constexpr int kL3Pf = 4;             // levels of StateRec prefetch per thread
constexpr int kL3Ring = 16384;       // recent state values kept in shared memory (power of two)
constexpr int kL3MaxLevels = 8192;   // level table cached in shared memory
constexpr int kLvPad = 2 * kL3Pf;      // empty levels padded on both sides of the level table
constexpr size_t kL3Smem = sizeof(double) * kL3Ring + sizeof(int) * (kL3MaxLevels + 1 + 2 * kLvPad);

__device__ __forceinline__ void l3_barrier(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// L3: grid 2*nb; even blocks forward (alpha), odd blocks backward (beta) of lattice b0 + blockIdx.x / 2.
// Level-synchronous: the states of a level only read states of earlier levels (later ones for beta), so
// each level is one parallel step and one barrier.  The values of the most recent kL3Ring states live in a
// shared-memory ring next to their global copy: slot s % kL3Ring holds state s while no state written since
// maps to the same slot, i.e. for alpha at level [lo, hi) every state s >= hi - kL3Ring (beta: s < lo +
// kL3Ring); older neighbours (long skip arcs) are read from global memory.  States with more than two arcs
// finish their LSE warp-cooperatively (ballot, then 32 arcs per round).  fp64 values, lse2f (K2's LSE).
__global__ void __launch_bounds__(kL3Threads) l3_forward_backward(Lat L, const StateRec* __restrict__ rec_f,
                                                                  const StateRec* __restrict__ rec_b,
                                                                  const float* __restrict__ w,
                                                                  double* __restrict__ alpha, double* __restrict__ beta,
                                                                  double* __restrict__ logp, float* __restrict__ losses,
                                                                  int b0) {
    extern __shared__ __align__(16) unsigned char l3_smem[];
    double* ring = reinterpret_cast<double*>(l3_smem);
    int* lv = reinterpret_cast<int*>(ring + kL3Ring);
    __shared__ int s_width;
    const int b = b0 + (blockIdx.x >> 1);
    const bool fwd = (blockIdx.x & 1) == 0;
    const int l0 = L.lvl_off[b], nlev = L.lvl_off[b + 1] - l0;
    const int s_start = L.state_off[b];
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned full = 0xffffffffu;
    const StateRec* rec = fwd ? rec_f : rec_b;
    double* val = fwd ? alpha : beta;
    const bool cached = nlev <= kL3MaxLevels;

    // Level table into shared memory and the widest level (decides how many warps take part).
    if (tid == 0) s_width = 0;
    __syncthreads();
    int wmax = 0;
    // lv[kLvPad + i] = level_off[l0 + i]; kLvPad empty levels of padding on both sides, so the prefetching
    // loop below runs whole groups of kL3Pf levels (and fetches kL3Pf ahead) without a bounds branch.
    for (int i = tid - kLvPad; i <= nlev + kLvPad; i += blockDim.x) {
        const int o = L.level_off[l0 + min(max(i, 0), nlev)];
        if (cached) lv[kLvPad + i] = o;
        if (i >= 0 && i < nlev) wmax = max(wmax, L.level_off[l0 + i + 1] - o);
    }
    atomicMax(&s_width, wmax);
    __syncthreads();
    const int width = s_width;
    const int nthr = max(32, min(kL3Threads, (width + 31) & ~31));
    if (tid >= nthr) return;
    auto level_lo = [&](int i) { return cached ? lv[kLvPad + i] : L.level_off[l0 + i]; };
    auto read_val = [&](int n, int lo, int hi) -> double {
        const bool in_ring = fwd ? (n >= hi - kL3Ring) : (n < lo + kL3Ring);
        return in_ring ? ring[n & (kL3Ring - 1)] : __ldcg(val + n);
    };
    auto extra_arc = [&](int k, int& n, float& wt) {
        if (fwd) {
            n = L.src[k];
            wt = w[k];
        } else {
            const int a = L.out_arc[k];
            n = L.dst[a];
            wt = w[a];
        }
    };
    // One state (or none, s >= hi) of level [lo, hi).
    auto do_state = [&](int s, int lo, int hi, const StateRec& r) {
        const bool on = s < hi;
        double acc = on ? static_cast<double>(r.init) : -INFINITY;
        if (on && r.deg > 0) acc = lse2f(acc, read_val(r.n0, lo, hi) + static_cast<double>(r.w0));
        if (on && r.deg > 1) acc = lse2f(acc, read_val(r.n1, lo, hi) + static_cast<double>(r.w1));
        unsigned heavy = __ballot_sync(full, on && r.deg > 2);
        while (heavy) {
            const int owner = __ffs(heavy) - 1;
            heavy &= heavy - 1;
            const int k0 = __shfl_sync(full, r.k0, owner), kend = __shfl_sync(full, r.kend, owner);
            double part = -INFINITY;
            for (int k = k0 + 2 + lane; k < kend; k += 32) {
                int n;
                float wt;
                extra_arc(k, n, wt);
                part = lse2f(part, read_val(n, lo, hi) + static_cast<double>(wt));
            }
            part = warp_lse(part);
            if (lane == owner) acc = lse2f(acc, part);
        }
        if (on) {
            ring[s & (kL3Ring - 1)] = acc;
            val[s] = acc;
        }
    };
    auto level_of = [&](int i) { return fwd ? i : nlev - 1 - i; };  // i-th processed level

    if (cached && width <= nthr) {
        // One state per thread and level: StateRecs fetched kPf levels ahead (register ring r[j] holds the
        // record of level i + j; it is refilled with level i + j + kPf right after use).
        const StateRec none{0, 0, -INFINITY, -INFINITY, 0, 0, -INFINITY, 0};
        const int* lvp = lv + kLvPad;  // lvp[-kLvPad .. nlev + kLvPad]
        auto fetch = [&](int i) -> StateRec {  // i < nlev + 2 kL3Pf; levels past the end are empty
            const int li = level_of(i);
            const int s = lvp[li] + tid;
            StateRec x = none;
            if (s < lvp[li + 1]) x = rec[s];
            return x;
        };
        StateRec r[kL3Pf];
#pragma unroll
        for (int j = 0; j < kL3Pf; ++j) r[j] = fetch(j);
        for (int i0 = 0; i0 < nlev; i0 += kL3Pf) {
#pragma unroll
            for (int j = 0; j < kL3Pf; ++j) {  // past nlev: empty levels (no state, a barrier)
                const int i = i0 + j;
                const int li = level_of(i);
                const int lo = lvp[li], hi = lvp[li + 1];
                do_state(lo + tid, lo, hi, r[j]);
                r[j] = fetch(i + kL3Pf);
                l3_barrier(nthr);
            }
        }
    } else {
        // Wide levels or very long lattices: strided over the level, no prefetch.
        for (int i = 0; i < nlev; ++i) {
            const int li = level_of(i);
            const int lo = level_lo(li), hi = level_lo(li + 1);
            for (int base = lo; base < hi; base += nthr) {
                const int s = base + tid;
                const StateRec rr = (s < hi) ? rec[s] : StateRec{0, 0, -INFINITY, -INFINITY, 0, 0, -INFINITY, 0};
                do_state(s, lo, hi, rr);
            }
            l3_barrier(nthr);
        }
    }
    if (!fwd && tid == 0) {
        const double lP = __ldcg(beta + s_start);
        logp[b] = lP;
        losses[b] = lP == INFINITY ? __int_as_float(0x7fc00000) : static_cast<float>(-lP);  // +inf: a NaN input
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
                                                     float* __restrict__ grads, int b0) {
    const int b = b0 + blockIdx.y;
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
                                               int Tmax, int Umax, int V, float* grads, bool vec4, int b0) {
    const int lane = threadIdx.x & 31;
    const int b = b0 + blockIdx.y;
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

// With a row index (row_off / row_arc: the arcs bound to each logits row, host-built) the gradient needs no
// float atomics, so it does not depend on scheduling (deterministic):
//   L4r  one thread per row: S[row] = sum of its arcs' occupancies, in row_arc order, and the first two arcs'
//        (v, occ) (rows with more are flagged)
//   L5r  warp per row: reads S and the (v, occ) pairs (one hop), issues the row's logit loads, stores
//        softmax * S with each arc's occ subtracted by the lane owning element v (the scatter, L6, is gone);
//        flagged rows walk their arcs 32 per warp pass.
__global__ void __launch_bounds__(256) l4_row_sums(Lat L, const float* __restrict__ w, const double* __restrict__ alpha,
                                                   const double* __restrict__ beta, const double* __restrict__ logp,
                                                   const int32_t* __restrict__ row_off,
                                                   const int32_t* __restrict__ row_arc, const int32_t* __restrict__ T_b,
                                                   const int32_t* __restrict__ U_b, int Tmax, int Umax,
                                                   float* __restrict__ rowS, float4* __restrict__ rowfix, int b0, int nb) {
    const int Up1 = Umax + 1;
    const int64_t cells = static_cast<int64_t>(Tmax) * Up1;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nb * cells;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = b0 + static_cast<int>(i / cells);
        const int r = static_cast<int>(i - (b - b0) * cells);
        const int t = r / Up1, u = r - t * Up1;
        const int64_t row = static_cast<int64_t>(b) * cells + r;
        const double lP = logp[b];
        float S = 0.f;
        // the row's arcs for L5r: (v0, occ0, v1, occ1) as bit patterns; v0 = -2: more than two arcs (generic)
        float4 fx = make_float4(__int_as_float(-1), 0.f, __int_as_float(-1), 0.f);
        if (t < T_b[b] && u <= U_b[b] && isfinite(lP)) {
            const int k0 = row_off[row], k1 = row_off[row + 1];
            for (int k = k0; k < k1; ++k) {
                const int a = row_arc[k];
                const float o = arc_occ(L, w, alpha, beta, lP, a);
                S += o;
                if (k == k0) fx = make_float4(__int_as_float(L.v[a]), o, fx.z, fx.w);
                if (k == k0 + 1) fx = make_float4(fx.x, fx.y, __int_as_float(L.v[a]), o);
            }
            if (k1 - k0 > 2) fx.x = __int_as_float(-2);
        }
        rowS[row] = S;
        rowfix[row] = fx;
    }
}

__global__ void __launch_bounds__(256) l5_rows_fused(const float* logits, const float* __restrict__ lse, Lat L,
                                                     const float* __restrict__ w, const double* __restrict__ alpha,
                                                     const double* __restrict__ beta, const float* __restrict__ rowS,
                                                     const float4* __restrict__ rowfix,
                                                     const int32_t* __restrict__ row_off,
                                                     const int32_t* __restrict__ row_arc, const int32_t* __restrict__ T_b,
                                                     const int32_t* __restrict__ U_b, const double* __restrict__ logp,
                                                     int Tmax, int Umax, int V, float* grads, bool vec4, int b0) {
    const int lane = threadIdx.x & 31;
    const int b = b0 + blockIdx.y;
    const int Up1 = Umax + 1;
    const int r = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (r >= Tmax * Up1) return;
    const int t = r / Up1, u = r - t * Up1;
    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    const double lP = logp[b];
    const bool live = t < T_b[b] && u <= U_b[b] && isfinite(lP);
    const float S = live ? rowS[row] : 0.f;
    const float l = live ? lse[row] : 0.f;
    const float* zr = logits + row * V;
    float* gr = grads + row * V;
    const bool on = live && S != 0.f && l != -INFINITY;
    const float ll = l * kLog2e;
    const int nv = V >> 2;
    float4 x[8];
    if (vec4) {  // the first chunk's loads go out before the arc fetches below
        const float4* z4 = reinterpret_cast<const float4*>(zr);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = j * 32 + lane;
            if (on && i < nv) x[j] = z4[i];
        }
    }
    const float4 fx = live ? rowfix[row] : make_float4(__int_as_float(-1), 0.f, __int_as_float(-1), 0.f);
    const int fv0 = __float_as_int(fx.x), fv1 = __float_as_int(fx.z);
    const bool generic = fv0 == -2;  // more than two bound arcs: the row index, 32 arcs per warp pass
    const int k0 = generic ? row_off[row] : 0, k1 = generic ? row_off[row + 1] : 0;
    const int a0 = (k0 + lane < k1) ? row_arc[k0 + lane] : -1;
    const int va0 = a0 >= 0 ? L.v[a0] : -1;
    const float oa0 = a0 >= 0 ? arc_occ(L, w, alpha, beta, lP, a0) : 0.f;
    // subtract the row's arcs' occupancies from the count (<= 4) elements [first, first + count) held in g
    auto sub_arcs = [&](float (&g)[4], int first, int count) {
        for (int kb = k0; kb < k1; kb += 32) {
            int va = va0;
            float oa = oa0;
            if (kb > k0) {  // rows with more than 32 bound arcs: later groups on the fly
                const int a = kb + lane < k1 ? row_arc[kb + lane] : -1;
                va = a >= 0 ? L.v[a] : -1;
                oa = a >= 0 ? arc_occ(L, w, alpha, beta, lP, a) : 0.f;
            }
            const int n = min(32, k1 - kb);
            for (int i = 0; i < n; ++i) {
                const int vi = __shfl_sync(0xffffffffu, va, i);
                const float oi = __shfl_sync(0xffffffffu, oa, i);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < count && vi == first + c) g[c] -= oi;
            }
        }
    };
    if (vec4) {
        const float4* z4 = reinterpret_cast<const float4*>(zr);
        float4* g4 = reinterpret_cast<float4*>(gr);
        for (int base = 0; base < nv; base += 256) {
            if (base > 0) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int i = base + j * 32 + lane;
                    if (on && i < nv) x[j] = z4[i];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = base + j * 32 + lane;
                float g[4] = {0.f, 0.f, 0.f, 0.f};
                if (on && i < nv) {
                    g[0] = ex2(fmaf(x[j].x, kLog2e, -ll)) * S;
                    g[1] = ex2(fmaf(x[j].y, kLog2e, -ll)) * S;
                    g[2] = ex2(fmaf(x[j].z, kLog2e, -ll)) * S;
                    g[3] = ex2(fmaf(x[j].w, kLog2e, -ll)) * S;
                }
                if (generic) {
                    sub_arcs(g, 4 * i, 4);  // warp-uniform condition
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (fv0 == 4 * i + c) g[c] -= fx.y;
                        if (fv1 == 4 * i + c) g[c] -= fx.w;
                    }
                }
                if (i < nv) g4[i] = make_float4(g[0], g[1], g[2], g[3]);
            }
        }
        return;
    }
    for (int i0 = 0; i0 < V; i0 += 32) {
        const int i = i0 + lane;
        float g[4] = {(on && i < V) ? ex2((zr[i] - l) * kLog2e) * S : 0.f, 0.f, 0.f, 0.f};
        if (generic) {
            sub_arcs(g, i, 1);
        } else {
            if (fv0 == i) g[0] -= fx.y;
            if (fv1 == i) g[0] -= fx.w;
        }
        if (i < V) gr[i] = g[0];
    }
}

}  // namespace

size_t lattice_workspace_bytes(int64_t B, int64_t Tmax, int64_t Umax, int64_t S, int64_t A) {
    const int64_t rows = B * Tmax * (Umax + 1);
    return align256(sizeof(float) * rows) * 2 + align256(sizeof(float) * A) + 2 * align256(sizeof(double) * S) +
           align256(sizeof(double) * B) + 2 * align256(sizeof(StateRec) * S) + align256(sizeof(float4) * rows);
}

}  // namespace rnnt

using rnnt::Lat;

extern "C" size_t rnnt_lattice_workspace_bytes(int B, int Tmax, int Umax, int num_states, int num_arcs) {
    if (B < 0 || Tmax < 1 || Umax < 0 || num_states < 0 || num_arcs < 0) return 0;
    return rnnt::lattice_workspace_bytes(B, Tmax, Umax, num_states, num_arcs);
}

// Launch schedule (as the loss path's, rnnt_api.cu): utterance chunks c; stream s runs L1(c) for every chunk,
// then per chunk [wait L3(c)] L4(c) L5(c) L6(c); the latency-bound L2 -> pack -> L3 of chunk c runs on
// aux[c] as soon as L1(c) is done, hidden under the bandwidth-bound L1 / L5 of the other chunks.
extern "C" rnnt_status rnnt_lattice_loss(const float* logits, const int32_t* logit_lens, const int32_t* target_lens,
                                         int B, int Tmax, int Umax, int V, const int32_t* state_off,
                                         const int32_t* lvl_off, const int32_t* level_off, const int32_t* in_off,
                                         const int32_t* out_off, const int32_t* out_arc, const int32_t* arc_src,
                                         const int32_t* arc_dst, const int32_t* arc_t, const int32_t* arc_u,
                                         const int32_t* arc_v, const float* final_w, const int32_t* row_off,
                                         const int32_t* row_arc, int num_states, int num_arcs,
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
    const int64_t cells = static_cast<int64_t>(Tmax) * (Umax + 1);
    const int64_t rows = static_cast<int64_t>(B) * cells;
    char* p = static_cast<char*>(workspace);
    auto take = [&](size_t bytes) {
        char* q = p;
        p += rnnt::align256(bytes);
        return q;
    };
    float* lse = reinterpret_cast<float*>(take(sizeof(float) * rows));
    float* rowS = reinterpret_cast<float*>(take(sizeof(float) * rows));
    float* w = reinterpret_cast<float*>(take(sizeof(float) * num_arcs));
    double* alpha = reinterpret_cast<double*>(take(sizeof(double) * num_states));
    double* beta = reinterpret_cast<double*>(take(sizeof(double) * num_states));
    double* logp = reinterpret_cast<double*>(take(sizeof(double) * B));
    auto* rec_f = reinterpret_cast<rnnt::StateRec*>(take(sizeof(rnnt::StateRec) * num_states));
    auto* rec_b = reinterpret_cast<rnnt::StateRec*>(take(sizeof(rnnt::StateRec) * num_states));
    auto* rowfix = reinterpret_cast<float4*>(take(sizeof(float4) * rows));  // row index path: 2 (v, occ) per row

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Lat L{state_off, lvl_off, level_off, in_off, out_off, out_arc, arc_src, arc_dst, arc_t, arc_u, arc_v,
                final_w};
    static thread_local int smem_set_dev = -1;  // the L3 shared-memory opt-in, once per device and thread
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return RNNT_ERR_CUDA;
    if (smem_set_dev != dev) {
        if (cudaFuncSetAttribute(rnnt::l3_forward_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(rnnt::kL3Smem)) != cudaSuccess)
            return RNNT_ERR_CUDA;
        smem_set_dev = dev;
    }
    const bool vec4 = V % 4 == 0 && reinterpret_cast<uintptr_t>(logits) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(grads) % 16 == 0;
    const int64_t bx = (cells + 7) / 8;

    int nch = rnnt::overlap_chunks(B, rows * V);
    rnnt::AuxPool* pool = (nch > 1) ? rnnt::aux_pool() : nullptr;
    if (pool == nullptr) nch = 1;
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    int cb0[rnnt::kMaxChunks + 1] = {0};
    for (int c = 0; c < nch; ++c) cb0[c + 1] = cb0[c] + B / nch + (c < B % nch ? 1 : 0);
    // Front half of chunk c: L1 on s, then L2 -> pack -> L3 on a (= s when sequential).
    for (int c = 0; c < nch; ++c) {
        const int b0 = cb0[c], nb = cb0[c + 1] - b0;
        cudaStream_t a = (nch > 1) ? pool->aux[c] : s;
        // L1: the log-softmax normalizer of every live row (K1 without the grid gathers).
        rnnt::Problem pr{logits + b0 * cells * V, nullptr, logit_lens + b0, target_lens + b0, nb, Tmax, Umax, V, 0,
                         rnnt::kRnnt, losses + b0, nullptr, nullptr, rnnt::kF32};
        rnnt::Workspace wk{lse + b0 * cells, nullptr, nullptr, nullptr, nullptr};  // lp == nullptr: lse only
        if (!ok(rnnt::launch_k1_lse_gather(pr, wk, s))) return RNNT_ERR_CUDA;
        if (nch > 1 && (!ok(cudaEventRecord(pool->k1_done[c], s)) || !ok(cudaStreamWaitEvent(a, pool->k1_done[c], 0))))
            return RNNT_ERR_CUDA;
        rnnt::l2_arc_weights<<<dim3(64, nb), 256, 0, a>>>(logits, lse, L, Tmax, Umax, V, w, b0);
        rnnt::l3_pack<<<dim3(32, nb), 256, 0, a>>>(L, w, rec_f, rec_b, b0);
        rnnt::l3_forward_backward<<<2 * nb, rnnt::kL3Threads, rnnt::kL3Smem, a>>>(L, rec_f, rec_b, w, alpha, beta, logp,
                                                                              losses, b0);
        if (nch > 1 && !ok(cudaEventRecord(pool->k2_done[c], a))) return RNNT_ERR_CUDA;
    }
    // Back half per chunk on s: with a row index, one fused row pass (L5'); without, L4 -> L5 -> L6.
    for (int c = 0; c < nch; ++c) {
        const int b0 = cb0[c], nb = cb0[c + 1] - b0;
        if (nch > 1 && !ok(cudaStreamWaitEvent(s, pool->k2_done[c], 0))) return RNNT_ERR_CUDA;
        if (!grads) continue;
        if (row_off) {
            rnnt::l4_row_sums<<<592, 256, 0, s>>>(L, w, alpha, beta, logp, row_off, row_arc, logit_lens, target_lens,
                                                  Tmax, Umax, rowS, rowfix, b0, nb);
            rnnt::l5_rows_fused<<<dim3(static_cast<unsigned>(bx), nb), 256, 0, s>>>(
                logits, lse, L, w, alpha, beta, rowS, rowfix, row_off, row_arc, logit_lens, target_lens, logp, Tmax,
                Umax, V, grads, vec4, b0);
            continue;
        }
        if (!ok(cudaMemsetAsync(rowS + b0 * cells, 0, sizeof(float) * nb * cells, s))) return RNNT_ERR_CUDA;
        const dim3 arc_grid(64, nb);
        rnnt::l46_occupancy<false><<<arc_grid, 256, 0, s>>>(L, w, alpha, beta, logp, Tmax, Umax, V, rowS, grads, b0);
        rnnt::l5_rows<<<dim3(static_cast<unsigned>(bx), nb), 256, 0, s>>>(logits, lse, rowS, logit_lens, target_lens,
                                                                         logp, Tmax, Umax, V, grads, vec4, b0);
        rnnt::l46_occupancy<true><<<arc_grid, 256, 0, s>>>(L, w, alpha, beta, logp, Tmax, Umax, V, rowS, grads, b0);
    }
    return cudaGetLastError() == cudaSuccess ? RNNT_OK : RNNT_ERR_CUDA;
}
