// k1_lse_gather.cu -- K1: log-softmax normalizer over V + Populate gather of the two arc weights per cell.
//
// PAPER.md §2.1 P:64 (the lattice weights are "RNN-T output log-probabilities", X = log_softmax(logits))
// and §2.2 P:88 / §2.3 P:92 (Populate = "indexed selection": every horizontal arc of the grid takes
// X[t,u,blank], every vertical arc X[t,u,y_{u+1}]).
//
// One warp per (b,t,u) row of V logits, streamed once from HBM with 128-bit loads (8 per lane in flight
// per chunk = 4 KB per warp), reduced with a lane-local online max/sum and a 5-step butterfly.  Exactly
// one ex2 per element.  Writes lse (fp32, row-major) and (X_blank, X_label) into the anti-diagonal-major
// lp array that the K2 wavefront reads coalesced.  Padded rows (t >= T_b or u > U_b) are skipped: never read.
#include "common.cuh"

namespace rnnt {
namespace {

constexpr int kUnroll = 8;  // float4 per lane per chunk

struct RowState {
    float m;   // lane-local running max
    float s;   // lane-local sum of 2^((x - m) * log2e)
    float zb;  // z[blank]  (valid on the owning lane only)
    float zy;  // z[y_u]    (valid on the owning lane only)
};

__device__ __forceinline__ void online_update(RowState& st, float cm, const float* xs, int n) {
    // cm = max(st.m, max xs): rescale the running sum, then accumulate this chunk.
    if (cm == -INFINITY) return;  // everything so far is -inf
    const float sc = (st.m == -INFINITY) ? 0.f : ex2((st.m - cm) * kLog2e);
    float acc = st.s * sc;
    const float cml = cm * kLog2e;
#pragma unroll
    for (int i = 0; i < n; ++i) acc += ex2(fmaf(xs[i], kLog2e, -cml));
    st.s = acc;
    st.m = cm;
}

__device__ __forceinline__ float pick4(const float4& v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

template <bool kVec>
__global__ void __launch_bounds__(kRowWarpsPerBlock * 32)
    k1_lse_gather(const float* __restrict__ logits, const int32_t* __restrict__ targets,
                  const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b, int B, int Tmax,
                  int Umax, int V, int blank, float* __restrict__ lse_out, float2* __restrict__ lp_out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowWarpsPerBlock + (threadIdx.x >> 5);
    const int Up1 = Umax + 1;
    const int64_t nrows = static_cast<int64_t>(B) * Tmax * Up1;
    if (row >= nrows) return;
    const int u = static_cast<int>(row % Up1);
    const int64_t bt = row / Up1;
    const int t = static_cast<int>(bt % Tmax);
    const int b = static_cast<int>(bt / Tmax);
    const int T = min(T_b[b], Tmax);
    const int U = min(U_b[b], Umax);
    if (t >= T || u > U) return;  // padding (or an invalid length, flagged by K2): never read

    int yv = -1;
    if (u < U) yv = targets[static_cast<int64_t>(b) * Umax + u];
    const bool ybad = (u < U) && (yv < 0 || yv >= V || yv == blank);
    if (ybad) yv = -1;

    RowState st{-INFINITY, 0.f, 0.f, 0.f};
    const float* zrow = logits + row * static_cast<int64_t>(V);

    if constexpr (kVec) {
        const float4* row4 = reinterpret_cast<const float4*>(zrow);
        const int nvec = V >> 2;
        const int bq = blank >> 2, yq = yv >> 2;  // float4 index holding blank / y
        for (int base = 0; base < nvec; base += 32 * kUnroll) {
            float4 x[kUnroll];
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) {
                const int i = base + j * 32 + lane;
                x[j] = (i < nvec) ? ld_stream_ro(row4 + i)
                                  : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
            float cm = st.m;
#pragma unroll
            for (int j = 0; j < kUnroll; ++j)
                cm = fmaxf(cm, fmaxf(fmaxf(x[j].x, x[j].y), fmaxf(x[j].z, x[j].w)));
            online_update(st, cm, reinterpret_cast<const float*>(x), 4 * kUnroll);
            // Populate gather: only the owning lane of the chunk holding blank / y picks its value.
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) {
                const int i = base + j * 32 + lane;
                if (i == bq) st.zb = pick4(x[j], blank & 3);
                if (i == yq) st.zy = pick4(x[j], yv & 3);
            }
        }
    } else {
        constexpr int kS = 4 * kUnroll;  // scalars per lane per chunk
        for (int base = 0; base < V; base += 32 * kS) {
            float x[kS];
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int i = base + j * 32 + lane;
                x[j] = (i < V) ? ld_stream_ro(zrow + i) : -INFINITY;
            }
            float cm = st.m;
#pragma unroll
            for (int j = 0; j < kS; ++j) cm = fmaxf(cm, x[j]);
            online_update(st, cm, x, kS);
#pragma unroll
            for (int j = 0; j < kS; ++j) {
                const int i = base + j * 32 + lane;
                if (i == blank) st.zb = x[j];
                if (i == yv) st.zy = x[j];
            }
        }
    }

    // Butterfly combine of (m, s); IEEE add/max are commutative so all lanes end bit-identical.
    float m = st.m, s = st.s;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
        const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
        const float M = fmaxf(m, m2);
        float acc = 0.f;
        if (M != -INFINITY) {
            if (m != -INFINITY) acc += s * ex2((m - M) * kLog2e);
            if (m2 != -INFINITY) acc += s2 * ex2((m2 - M) * kLog2e);
        }
        m = M;
        s = acc;
    }
    // Fetch the gathered values from their owning lanes.
    const int owner_b = kVec ? ((blank >> 2) & 31) : (blank & 31);
    const float zb = __shfl_sync(0xffffffffu, st.zb, owner_b);
    const int owner_y = (yv < 0) ? 0 : (kVec ? ((yv >> 2) & 31) : (yv & 31));
    const float zy = __shfl_sync(0xffffffffu, st.zy, owner_y);

    if (lane == 0) {
        const float lse = (m == -INFINITY) ? -INFINITY : m + lg2(s) * kLn2;
        lse_out[row] = lse;
        float xb, xy;
        if (lse == -INFINITY) {  // an all -inf row forbids its arcs (reading R12)
            xb = -INFINITY;
            xy = -INFINITY;
        } else {
            xb = zb - lse;
            xy = (u < U) ? (ybad ? __int_as_float(0x7fc00000) : zy - lse) : -INFINITY;
        }
        const int64_t diag = static_cast<int64_t>(b) * (Tmax + Umax) + (t + u);
        lp_out[diag * Up1 + u] = make_float2(xb, xy);
    }
}

}  // namespace

cudaError_t launch_k1_lse_gather(const Problem& p, const Workspace& w, cudaStream_t s) {
    const int64_t nrows = static_cast<int64_t>(p.B) * p.Tmax * (p.Umax + 1);
    const int64_t blocks = (nrows + kRowWarpsPerBlock - 1) / kRowWarpsPerBlock;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const bool vec = (p.V % 4 == 0) && (reinterpret_cast<uintptr_t>(p.logits) % 16 == 0);
    if (vec)
        k1_lse_gather<true><<<static_cast<unsigned>(blocks), kRowWarpsPerBlock * 32, 0, s>>>(
            p.logits, p.targets, p.T_b, p.U_b, p.B, p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
    else
        k1_lse_gather<false><<<static_cast<unsigned>(blocks), kRowWarpsPerBlock * 32, 0, s>>>(
            p.logits, p.targets, p.T_b, p.U_b, p.B, p.Tmax, p.Umax, p.V, p.blank, w.lse, w.lp);
    return cudaGetLastError();
}

}  // namespace rnnt
