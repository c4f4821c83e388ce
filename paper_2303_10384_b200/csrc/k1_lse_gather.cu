// k1_lse_gather.cu -- K1: log-softmax normalizer over V + Populate gather of the two arc weights per cell.
//
// PAPER.md §2.1 P:64 (the lattice weights are "RNN-T output log-probabilities", X = log_softmax(logits))
// and §2.2 P:88 / §2.3 P:92 (Populate = "indexed selection": every horizontal arc of the grid takes
// X[t,u,blank], every vertical arc X[t,u,y_{u+1}]).
//
// Rows of V logits are streamed once from HBM with 128-bit loads under an L2 evict-first policy (so the
// workspace the next kernels reuse stays in L2).  Wide rows: one warp per (b,t,u) row, 32 elements per lane
// per chunk (k1_lse_gather_w).  Narrow rows (fp32 V <= 512, 16-bit V <= 512): a group of G = 4..16 lanes
// per row with 8 x 128-bit loads per lane, so a warp still keeps 4 KB in flight (k1_lse_gather_g).  Per lane: max over the chunk (FMNMX3), then one ex2 per element with packed
// FFMA2/FADD2 around it; across chunks a lane-local online rescale; across the G lanes one max-reduce,
// one rescale, one sum-reduce (xor butterflies stay inside the group).  16-bit logits are widened to fp32
// in registers (half-precision populate, fp32/fp64 scores).  The two gathered logits are fetched
// by the group's lanes 0 / 1 with scalar loads that merge in L2 with the row's loads.  Writes lse (fp32,
// row-major) and (X_blank, X_label) into the anti-diagonal-major lp array that the K2 wavefront reads.
// Padded rows (t >= T_b or u > U_b) are never read.
#include "common.cuh"
#include "elem.cuh"

namespace rnnt {
namespace {

constexpr int kPerLane = 32;  // elements per lane per chunk

template <typename Z, bool kVec, typename VecT = uint4>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32, 4)
    k1_lse_gather_w(const Z* __restrict__ logits, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int b0, int Tmax, int Umax,
                  int V, int blank, float* __restrict__ lse_out, double2* __restrict__ lp_out) {
    const int lane = threadIdx.x & 31;
    const int b = b0 + static_cast<int>(blockIdx.y);
    const int Up1 = Umax + 1;
    const int r = static_cast<int>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5);  // row in utterance
    if (r >= Tmax * Up1) return;
    const int t = r / Up1;
    const int u = r - t * Up1;
    const int T = min(T_b[b], Tmax);
    const int U = min(U_b[b], Umax);
    if (t >= T || u > U) return;  // padding (or an invalid length, flagged by K2): never read

    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    const Z* zrow = logits + row * static_cast<int64_t>(V);
    constexpr int E = static_cast<int>(sizeof(VecT) / sizeof(Z)), kU = kPerLane / E;
    const uint64_t pol = l2_evict_first();
    const VecT* row4 = reinterpret_cast<const VecT*>(zrow);
    const int nvec = V / E;
    VecT raw[kU];
    // 16-bit rows: the first chunk goes out before anything that depends on other loads (measured: K1 bf16
    // 0.95 -> 0.88 ms).  fp32 rows keep the loads after the gather (the early issue costs fp32 28 registers
    // and a quarter of its occupancy: measured slower).
    constexpr bool kEarly = kVec && sizeof(Z) == 2;
    if constexpr (kEarly) {
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int i = j * 32 + lane;
            raw[j] = (i < nvec) ? ldv_ro(row4 + i, pol) : zero_vec<VecT>();
        }
    }

    int yv = -1;
    if (u < U && targets) yv = targets[static_cast<int64_t>(b) * Umax + u];
    const bool ybad = targets && (u < U) && (yv < 0 || yv >= V || yv == blank);
    if (ybad) yv = -1;
    // Populate gather: lanes 0 / 1 fetch z[blank] / z[y] with scalar loads issued alongside the row's
    // loads (same sectors, merged in L2: no extra DRAM traffic, no register indexing).
    float zb = 0.f, zy = 0.f;
    if (lane == 0) zb = lds_scalar(zrow + blank);
    if (lane == 1 && yv >= 0) zy = lds_scalar(zrow + yv);

    float m = -INFINITY;  // lane-local running max
    float s = 0.f;        // lane-local sum of e^(x - m)
    const f32x2 l2e = pk(kLog2e, kLog2e);
    auto absorb = [&](const float (&x)[kPerLane]) {  // online max / sum-exp update with one chunk
        float cm = m;
#pragma unroll
        for (int i = 0; i < kPerLane; i += 2) cm = max3(cm, x[i], x[i + 1]);
        if (cm == -INFINITY) return;
        const float sc = (m == -INFINITY) ? 0.f : ex2((m - cm) * kLog2e);
        const f32x2 nml = pk(-cm * kLog2e, -cm * kLog2e);
        f32x2 acc0 = pk(0.f, 0.f), acc1 = pk(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < kPerLane; i += 4) {
            acc0 = fadd2(acc0, ex2x2(ffma2(pk(x[i], x[i + 1]), l2e, nml)));
            acc1 = fadd2(acc1, ex2x2(ffma2(pk(x[i + 2], x[i + 3]), l2e, nml)));
        }
        const float2 a = upk(fadd2(acc0, acc1));
        s = fmaf(s, sc, a.x + a.y);
        m = cm;
    };

    if constexpr (kVec) {
        for (int base = 0; base < nvec; base += 32 * kU) {
            if (!kEarly || base > 0) {
#pragma unroll
                for (int j = 0; j < kU; ++j) {
                    const int i = base + j * 32 + lane;
                    raw[j] = (i < nvec) ? ldv_ro(row4 + i, pol) : zero_vec<VecT>();
                }
            }
            float x[kPerLane];
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                float f[E];
                Elem<Z>::unpack(raw[j], f);
                const bool in = base + j * 32 + lane < nvec;
#pragma unroll
                for (int e = 0; e < E; ++e) x[j * E + e] = in ? f[e] : -INFINITY;
            }
            absorb(x);
        }
    } else {
        for (int base = 0; base < V; base += 32 * kPerLane) {
            float x[kPerLane];
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = base + j * 32 + lane;
                x[j] = (i < V) ? lds_scalar(zrow + i) : -INFINITY;
            }
            absorb(x);
        }
    }

    // Warp combine: M = max over lanes; S = sum over lanes of s * e^(m - M).  Butterflies leave every lane
    // with bit-identical M and S (IEEE max/add are commutative), independent of grid shape.
    float M = m;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float S = (m == -INFINITY) ? 0.f : s * ex2((m - M) * kLog2e);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
    zb = __shfl_sync(0xffffffffu, zb, 0);
    zy = __shfl_sync(0xffffffffu, zy, 1);

    if (lane == 0) {
        const float lse = (M == -INFINITY) ? -INFINITY : M + lg2(S) * kLn2;
        lse_out[row] = lse;
        float xb, xy;
        if (lse == -INFINITY) {  // an all -inf row forbids its arcs (reading R12)
            xb = -INFINITY;
            xy = -INFINITY;
        } else if (lse != lse) {  // a NaN in the row: +inf arc scores (common.cuh kNanArc)
            xb = INFINITY;
            xy = (u < U) ? INFINITY : -INFINITY;
        } else {
            xb = zb - lse;
            xy = (u < U) ? (ybad ? __int_as_float(0x7fc00000) : zy - lse) : -INFINITY;
        }
        const int64_t diag = static_cast<int64_t>(b) * (Tmax + Umax) + (t + u);
        if (lp_out) lp_out[diag * Up1 + u] = make_double2(xb, xy);
    }
}


// 16-bit wide rows, two rows per warp (k1_lse_gather_w2): a warp loads the first chunk of both its rows
// before anything else, then finishes the two rows with interleaved reductions (independent chains), halving
// the per-row overhead (index math, gathers, butterflies, stores) per byte.  Measured c3 bf16: 0.882 ->
// 0.865 ms (A/B); slots past V set to -inf vectors instead of a per-element select: 0.862 -> 0.808 ms, and
// only in a partial chunk (no default fill of the load registers): -> 0.753 ms.
template <typename Z, typename VecT>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32, 3)
    k1_lse_gather_w2(const Z* __restrict__ logits, const int32_t* __restrict__ targets,
                     const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int b0, int Tmax, int Umax,
                     int V, int blank, float* __restrict__ lse_out, double2* __restrict__ lp_out) {
    constexpr int E = static_cast<int>(sizeof(VecT) / sizeof(Z)), kU = kPerLane / E;
    const int lane = threadIdx.x & 31;
    const int b = b0 + static_cast<int>(blockIdx.y);
    const int Up1 = Umax + 1;
    const int r0 = (static_cast<int>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5)) * 2;
    const int T = min(T_b[b], Tmax);
    const int U = min(U_b[b], Umax);
    int tt[2], uu[2];
    bool live[2];
    tt[0] = r0 / Up1;  // one division per warp: row r0 + 1 is the next cell of the same or the next frame
    uu[0] = r0 - tt[0] * Up1;
    const bool wrap = uu[0] + 1 == Up1;
    tt[1] = tt[0] + (wrap ? 1 : 0);
    uu[1] = wrap ? 0 : uu[0] + 1;
#pragma unroll
    for (int k = 0; k < 2; ++k)
        live[k] = r0 + k < Tmax * Up1 && tt[k] < T && uu[k] <= U;  // padding rows are never read
    if (!live[0] && !live[1]) return;
    const int64_t row0 = static_cast<int64_t>(b) * Tmax * Up1 + r0;
    const uint64_t pol = l2_evict_first();
    const int nvec = V / E;
    const VecT* row4[2] = {reinterpret_cast<const VecT*>(logits + row0 * static_cast<int64_t>(V)),
                            reinterpret_cast<const VecT*>(logits + (row0 + 1) * static_cast<int64_t>(V))};
    VecT raw[2][kU];
    // loads only where in range (no default register fill); a partial chunk gets its -inf slots afterwards
    auto load_chunk = [&](int base) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                const int i = base + j * 32 + lane;
                if (live[k] && i < nvec) raw[k][j] = ldv_ro(row4[k] + i, pol);
            }
        if (base + 32 * kU > nvec) {  // warp-uniform: only a last, partial chunk
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int j = 0; j < kU; ++j)
                    if (base + j * 32 + lane >= nvec) raw[k][j] = neg_inf_vec<Z, VecT>();
        }
    };
    load_chunk(0);
    int yv[2];
    bool ybad[2];
    float zb[2] = {0.f, 0.f}, zy[2] = {0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        yv[k] = (live[k] && uu[k] < U && targets) ? targets[static_cast<int64_t>(b) * Umax + uu[k]] : -1;
        ybad[k] = targets && (uu[k] < U) && (yv[k] < 0 || yv[k] >= V || yv[k] == blank);
        if (ybad[k]) yv[k] = -1;
        const Z* zrow = logits + (row0 + k) * static_cast<int64_t>(V);
        if (live[k] && lane == 0) zb[k] = lds_scalar(zrow + blank);
        if (live[k] && lane == 1 && yv[k] >= 0) zy[k] = lds_scalar(zrow + yv[k]);
    }
    float m[2] = {-INFINITY, -INFINITY}, sacc[2] = {0.f, 0.f};
    const f32x2 l2e = pk(kLog2e, kLog2e);
    auto absorb = [&](int k, const float (&x)[kPerLane]) {
        float cm = m[k];
#pragma unroll
        for (int i = 0; i < kPerLane; i += 2) cm = max3(cm, x[i], x[i + 1]);
        if (cm == -INFINITY) return;
        const float sc = (m[k] == -INFINITY) ? 0.f : ex2((m[k] - cm) * kLog2e);
        const f32x2 nml = pk(-cm * kLog2e, -cm * kLog2e);
        f32x2 acc0 = pk(0.f, 0.f), acc1 = pk(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < kPerLane; i += 4) {
            acc0 = fadd2(acc0, ex2x2(ffma2(pk(x[i], x[i + 1]), l2e, nml)));
            acc1 = fadd2(acc1, ex2x2(ffma2(pk(x[i + 2], x[i + 3]), l2e, nml)));
        }
        const float2 a2 = upk(fadd2(acc0, acc1));
        sacc[k] = fmaf(sacc[k], sc, a2.x + a2.y);
        m[k] = cm;
    };
    for (int base = 0; base < nvec; base += 32 * kU) {
        if (base > 0) load_chunk(base);
        // slots past V were loaded as -inf vectors: no per-element select
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float x[kPerLane];
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                float f[E];
                Elem<Z>::unpack(raw[k][j], f);
#pragma unroll
                for (int e = 0; e < E; ++e) x[j * E + e] = f[e];
            }
            if (live[k]) absorb(k, x);
        }
    }
    float M[2] = {m[0], m[1]};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        M[0] = fmaxf(M[0], __shfl_xor_sync(0xffffffffu, M[0], off));
        M[1] = fmaxf(M[1], __shfl_xor_sync(0xffffffffu, M[1], off));
    }
    float S[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) S[k] = (m[k] == -INFINITY) ? 0.f : sacc[k] * ex2((m[k] - M[k]) * kLog2e);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        S[0] += __shfl_xor_sync(0xffffffffu, S[0], off);
        S[1] += __shfl_xor_sync(0xffffffffu, S[1], off);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        zb[k] = __shfl_sync(0xffffffffu, zb[k], 0);
        zy[k] = __shfl_sync(0xffffffffu, zy[k], 1);
    }
    const bool wr = (lane == 0 && live[0]) || (lane == 1 && live[1]);
    if (wr) {  // lane k writes row k
        const int k = lane;
        const float Mk = k ? M[1] : M[0], Sk = k ? S[1] : S[0];
        const float lse = (Mk == -INFINITY) ? -INFINITY : Mk + lg2(Sk) * kLn2;
        lse_out[row0 + k] = lse;
        float xb, xy;
        const int t = k ? tt[1] : tt[0], u = k ? uu[1] : uu[0];
        if (lse == -INFINITY) {  // an all -inf row forbids its arcs (reading R12)
            xb = -INFINITY;
            xy = -INFINITY;
        } else if (lse != lse) {  // a NaN in the row: +inf arc scores (common.cuh kNanArc)
            xb = INFINITY;
            xy = (u < U) ? INFINITY : -INFINITY;
        } else {
            xb = (k ? zb[1] : zb[0]) - lse;
            xy = (u < U) ? ((k ? ybad[1] : ybad[0]) ? __int_as_float(0x7fc00000) : (k ? zy[1] : zy[0]) - lse)
                         : -INFINITY;
        }
        const int64_t diag = static_cast<int64_t>(b) * (Tmax + Umax) + (t + u);
        if (lp_out) lp_out[diag * Up1 + u] = make_double2(xb, xy);
    }
}

constexpr int kVecPerLane = 8;  // 128-bit loads per lane per chunk

template <typename Z, int G, typename VecT = uint4>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32)
    k1_lse_gather_g(const Z* __restrict__ logits, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int b0, int Tmax, int Umax,
                  int V, int blank, float* __restrict__ lse_out, double2* __restrict__ lp_out) {
    constexpr int E = static_cast<int>(sizeof(VecT) / sizeof(Z)), kU = kVecPerLane, kRowsPerWarp = 32 / G;
    const int lane = threadIdx.x & 31;
    const int sl = lane & (G - 1);  // lane within the row group
    const int b = b0 + static_cast<int>(blockIdx.y);
    const int Up1 = Umax + 1;
    const int r = (static_cast<int>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5)) * kRowsPerWarp + lane / G;
    const int t = r / Up1;
    const int u = r - t * Up1;
    const int T = min(T_b[b], Tmax);
    const int U = min(U_b[b], Umax);
    // A group whose row is padding (or beyond the grid) loads nothing and stores nothing, but still takes
    // part in the warp's shuffles.
    const bool live = (r < Tmax * Up1) && (t < T) && (u <= U);
    if (__all_sync(0xffffffffu, !live)) return;

    int yv = -1;
    if (live && u < U && targets) yv = targets[static_cast<int64_t>(b) * Umax + u];
    const bool ybad = targets && (u < U) && (yv < 0 || yv >= V || yv == blank);
    if (ybad) yv = -1;

    const int64_t row = static_cast<int64_t>(b) * Tmax * Up1 + r;
    const Z* zrow = logits + row * static_cast<int64_t>(V);
    const VecT* row4 = reinterpret_cast<const VecT*>(zrow);
    const uint64_t pol = l2_evict_first();
    // Populate gather: lanes 0 / 1 of the group fetch z[blank] / z[y] with scalar loads issued alongside the
    // row's loads (same sectors, merged in L2: no extra DRAM traffic, no register indexing).
    float zb = 0.f, zy = 0.f;
    if (live && sl == 0) zb = lds_scalar(zrow + blank);
    if (live && sl == 1 && yv >= 0) zy = lds_scalar(zrow + yv);

    const int nvec = V / E;
    const f32x2 l2e = pk(kLog2e, kLog2e);
    float m = -INFINITY;  // lane-local running max
    float s = 0.f;        // lane-local sum of e^(x - m)
    for (int base = 0; base < nvec; base += G * kU) {
        VecT raw[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int i = base + j * G + sl;
            raw[j] = (live && i < nvec) ? ldv_ro(row4 + i, pol) : zero_vec<VecT>();
        }
        // Only a partial last chunk needs -inf fill for the slots past V (warp-uniform condition).
        const bool partial = base + G * kU > nvec;
        // Pass 1: chunk max (widening 16-bit values on the fly).
        float cm = m;
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            float f[E];
            Elem<Z>::unpack(raw[j], f);
            if (partial && base + j * G + sl >= nvec) {
#pragma unroll
                for (int e = 0; e < E; ++e) f[e] = -INFINITY;
            }
#pragma unroll
            for (int e = 0; e < E; e += 2) cm = max3(cm, f[e], f[e + 1]);
        }
        if (cm == -INFINITY) continue;
        // Pass 2: sum of 2^((x - cm) log2 e), rescaling the running sum once.
        const float sc = (m == -INFINITY) ? 0.f : ex2((m - cm) * kLog2e);
        const f32x2 nml = pk(-cm * kLog2e, -cm * kLog2e);
        f32x2 acc0 = pk(0.f, 0.f), acc1 = pk(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            float f[E];
            Elem<Z>::unpack(raw[j], f);
            if (partial && base + j * G + sl >= nvec) {
#pragma unroll
                for (int e = 0; e < E; ++e) f[e] = -INFINITY;
            }
#pragma unroll
            for (int e = 0; e < E; e += 4) {
                acc0 = fadd2(acc0, ex2x2(ffma2(pk(f[e], f[e + 1]), l2e, nml)));
                acc1 = fadd2(acc1, ex2x2(ffma2(pk(f[e + 2], f[e + 3]), l2e, nml)));
            }
        }
        const float2 a = upk(fadd2(acc0, acc1));
        s = fmaf(s, sc, a.x + a.y);
        m = cm;
    }

    // Group combine: M = max over the G lanes; S = sum of s * e^(m - M).  Xor butterflies with offsets < G
    // stay inside the group and leave every lane bit-identical (IEEE max/add are commutative).
    float M = m;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float S = (m == -INFINITY) ? 0.f : s * ex2((m - M) * kLog2e);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
    const int g0 = lane & ~(G - 1);
    zb = __shfl_sync(0xffffffffu, zb, g0);
    zy = __shfl_sync(0xffffffffu, zy, g0 + 1);

    if (live && sl == 0) {
        const float lse = (M == -INFINITY) ? -INFINITY : M + lg2(S) * kLn2;
        lse_out[row] = lse;
        float xb, xy;
        if (lse == -INFINITY) {  // an all -inf row forbids its arcs (reading R12)
            xb = -INFINITY;
            xy = -INFINITY;
        } else if (lse != lse) {  // a NaN in the row: +inf arc scores (common.cuh kNanArc)
            xb = INFINITY;
            xy = (u < U) ? INFINITY : -INFINITY;
        } else {
            xb = zb - lse;
            xy = (u < U) ? (ybad ? __int_as_float(0x7fc00000) : zy - lse) : -INFINITY;
        }
        const int64_t diag = static_cast<int64_t>(b) * (Tmax + Umax) + (t + u);
        if (lp_out) lp_out[diag * Up1 + u] = make_double2(xb, xy);
    }
}

template <typename Z, int G, typename VecT = uint4>
void launch_g(const Problem& p, const Workspace& w, cudaStream_t s, const Z* z, int64_t rows_per_utt) {
    constexpr int kRowsPerBlock = kRowWarpsPerBlock * (32 / G);
    const int64_t bx = (rows_per_utt + kRowsPerBlock - 1) / kRowsPerBlock;
    for (int b0 = 0; b0 < p.B; b0 += 65535) {
        const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(min(65535, p.B - b0)));
        k1_lse_gather_g<Z, G, VecT><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(z, p.targets, p.T_b, p.U_b, b0, p.Tmax,
                                                                       p.Umax, p.V, p.blank, w.lse, w.lp);
    }
}

}  // namespace

// Lanes per row for the grouped kernels: the smallest power of two in [4, 32] whose 8-vector-per-lane
// chunk covers the row (32 = use the one-warp-per-row kernels).
int lanes_per_row(int nvec) {
    int g = 4;
    while (g < 32 && g * kVecPerLane < nvec) g *= 2;
    return g;
}

namespace {

template <typename Z>
cudaError_t launch_t(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int64_t rows_per_utt = static_cast<int64_t>(p.Tmax) * (p.Umax + 1);
    if (rows_per_utt > 0x7fffffffLL / 2) return cudaErrorInvalidConfiguration;
    const Z* z = static_cast<const Z*>(p.logits);
    constexpr int E = Elem<Z>::kPerVec;
    const bool vec = (p.V % E == 0) && (reinterpret_cast<uintptr_t>(z) % 16 == 0);
    const int g = vec ? lanes_per_row(p.V / E) : 32;
    // Widest row group: 16 lanes for fp32 (rows of <= 512 elements: p124's V = 500 K1 0.435 -> 0.338 ms),
    // 8 for 16-bit storage (16-lane groups measured slower than the two-rows-per-warp kernel: bf16 c3 1.09 vs
    // 0.88 ms).
    constexpr int gmax = sizeof(Z) == 4 ? 16 : 8;
    if (g <= gmax) {  // narrow rows: grouped kernel
        switch (g) {
            case 4: launch_g<Z, 4>(p, w, s, z, rows_per_utt); break;
            case 8: launch_g<Z, 8>(p, w, s, z, rows_per_utt); break;
            default: launch_g<Z, 16>(p, w, s, z, rows_per_utt); break;
        }
        return cudaGetLastError();
    }
    if constexpr (sizeof(Z) == 2) {  // 16-bit wide rows: two rows per warp, 128-bit or (V % 8 == 4) 64-bit loads
      const bool vec8 = (p.V % 4 == 0) && (reinterpret_cast<uintptr_t>(z) % 8 == 0);
      const int g8 = (!vec && vec8) ? lanes_per_row(p.V / 4) : 32;
      if (g8 < 32) {  // narrow 64-bit rows (e.g. V = 500): row groups, 8 x 64-bit loads per lane
        switch (g8) {
            case 4: launch_g<Z, 4, uint2>(p, w, s, z, rows_per_utt); break;
            case 8: launch_g<Z, 8, uint2>(p, w, s, z, rows_per_utt); break;
            default: launch_g<Z, 16, uint2>(p, w, s, z, rows_per_utt); break;
        }
        return cudaGetLastError();
      }
      if (vec || vec8) {
        const int64_t bx2 = (rows_per_utt + 2 * kRowWarpsPerBlock - 1) / (2 * kRowWarpsPerBlock);
        for (int b0 = 0; b0 < p.B; b0 += 65535) {
            const dim3 grid(static_cast<unsigned>(bx2), static_cast<unsigned>(min(65535, p.B - b0)));
            if (vec)
                k1_lse_gather_w2<Z, uint4><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(z, p.targets, p.T_b, p.U_b, b0,
                                                                                p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
            else
                k1_lse_gather_w2<Z, uint2><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(z, p.targets, p.T_b, p.U_b, b0,
                                                                                p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
        }
        return cudaGetLastError();
      }
    }
    const bool vec2 = !vec && sizeof(Z) == 4 && (p.V % 2 == 0) && (reinterpret_cast<uintptr_t>(z) % 8 == 0);
    const int64_t bx = (rows_per_utt + kRowWarpsPerBlock - 1) / kRowWarpsPerBlock;
    for (int b0 = 0; b0 < p.B; b0 += 65535) {
        const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(min(65535, p.B - b0)));
        if (vec2)  // fp32 rows with V % 4 == 2: 64-bit vectors
            k1_lse_gather_w<Z, true, uint2><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
        else if (vec)
            k1_lse_gather_w<Z, true><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
        else
            k1_lse_gather_w<Z, false><<<grid, kRowWarpsPerBlock * 32, 0, s>>>(
                z, p.targets, p.T_b, p.U_b, b0, p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_k1_lse_gather(const Problem& p, const Workspace& w, cudaStream_t s) {
    switch (p.dtype) {
        case kF32: return launch_t<float>(p, w, s);
        case kF16: return launch_t<__half>(p, w, s);
        case kBF16: return launch_t<__nv_bfloat16>(p, w, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace rnnt
