// k7_joint_grad.cu -- the backward of the fused joint network + loss (training).
//
// Gradients of sum_b loss_b with respect to the joint's inputs (readings R22, R23):
//   dz(t,u,v)  = softmax(z)(v) (occ_b + occ_y) - [v = blank] occ_b - [v = y_u] occ_y      (K3's formula)
//   dh(t,u,:)  = sum_v dz(t,u,v) W(v,:)                  dW(v,:) = sum_{t,u} dz(t,u,v) h(t,u,:)
//   dbias(v)   = sum_{t,u} dz(t,u,v)
//   dpre       = dh * (1 - h^2)   (dh accumulated in fp32 in TMEM, stored in bf16; tanh' from the stored bf16 h)
//   d enc(b,t,:) = sum_{u <= U_b} dpre(t,u,:)           d pred(b,u,:) = sum_{t < T_b} dpre(t,u,:)
// over the valid cells.  Pipeline (all on the caller's stream, every kernel this library's own):
//   K6 (forward: lse, gathers, and h from its builders' registers) -> K2 (alpha, beta, losses) -> K6<grad>
//   (k6_dz_2sm: z again on the tensor cores from the stored h, its epilogue writes dz in bf16) -> K8 (dh = dz W,
//   CTA-pair tcgen05 GEMM) and K9
//   (dW = dz^T h and dbias, CTA-pair tcgen05 GEMM split over row ranges, k9_reduce) (k8_joint_bwd.cu) -> K7
//   (tanh' and the two reductions, one streaming pass over dh and h).  The [B,T,U+1,V] logits never exist; dz
//   does, in
//   bf16 (half the bytes of fp32 logits), because dW needs it against every row and dh against every v, and a
//   128-row tile's fp32 dh (128 x H) alone fills TMEM at H = 512.  Rows are the compact valid
//   cells (K6's row map); with the caller's valid-row count the GEMMs cover exactly those, else the padded row
//   count B*Tmax*(Umax+1) with the tail rows zeroed.
#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "elem.cuh"
#include "joint.cuh"
#include "rnnt_b200.h"
#include "tc.cuh"

namespace rnnt {
namespace {

// Zero rows [*nrows, R) of dz ([R][Vp]) and h ([R][Hg]) so the padded-row GEMMs see no stale data.
__global__ void __launch_bounds__(256) k7_zero_tail(const int* __restrict__ nrows, int64_t R, int Vp, int Hg,
                                                    __nv_bfloat16* dz, __nv_bfloat16* h) {
    const int64_t r0 = *nrows;
    const int64_t nz = (R - r0) * Vp / 8, nh = (R - r0) * Hg / 8;  // 16-byte units
    uint4* z4 = reinterpret_cast<uint4*>(dz + r0 * Vp);
    uint4* h4 = reinterpret_cast<uint4*>(h + r0 * Hg);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nz + nh;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < nz)
            z4[i] = make_uint4(0u, 0u, 0u, 0u);
        else
            h4[i - nz] = make_uint4(0u, 0u, 0u, 0u);
    }
}

// valid_rows given by the caller must equal the row map's count; else every loss is NaN (loud failure: the
// GEMMs ran over the wrong rows).
__global__ void k7_check_rows(const int* __restrict__ nrows, int64_t valid_rows, int B, float* __restrict__ losses) {
    if (*nrows == valid_rows) return;
    for (int i = threadIdx.x; i < B; i += blockDim.x) losses[i] = __int_as_float(0x7fc00000);
}

__device__ __forceinline__ int utt_count(const int32_t* T_b, const int32_t* U_b, int i, int Tmax, int Umax) {
    const int T = T_b[i], U = U_b[i];
    return (T >= 1 && T <= Tmax && U >= 0 && U <= Umax) ? T * (U + 1) : 0;
}

// First compact row of utterance b (the row map's order): a block-wide sum of the earlier counts.
__device__ int utt_offset(const int32_t* T_b, const int32_t* U_b, int b, int Tmax, int Umax, int* s_part) {
    int part = 0;
    for (int i = threadIdx.x; i < b; i += blockDim.x) part += utt_count(T_b, U_b, i, Tmax, Umax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) off += s_part[w];
    return off;
}

// K7, pass 1: block (chunk, b, slice) takes frames [chunk * kTC, +kTC) of utterance b and a 256-column slice of
// H, and streams each of its rows of dh (K8's output) and h ONCE: dpre = dh * (1 - h^2) (kPre: the input already
// is dpre, K8 applied tanh'; h is not read).  256 threads = 8 warps; lane = 8 columns, so a warp reads a whole
// 512-byte row segment per 16-byte load; warp w owns units u = w (mod 8) and loads its kTC frames of a unit at
// once.  Its sum over the chunk's frames is the chunk's partial of d pred(b, u) (-> part); its contribution to
// d enc(b, t) stays in registers and the 8 warps' partials are added in a fixed tree order through shared
// memory (the block owns every unit of its frames: d enc is complete, written directly).  (Two blocks per SM
// at <= 128 registers, with fewer frames in flight per warp, was slower: 0.83 vs 0.63 ms at c3.)  Pass 2 sums the
// chunk partials of d pred in chunk order.  Deterministic.
constexpr int kTC = 8;
// K9's SM cap when K7 runs beside it (K7 fills the rest).  0 = sequential (the default): A/B on B200, 3
// alternating reps of 60-step training steps (scripts/gpu_k9ovl2.sh): c3 7.29 ms sequential, 7.19 with K9 on
// 96 SMs, 7.25 on 112; p124 2.13 sequential, 2.14 / 2.16 -- within the power-capped clock's noise, so the
// simpler schedule stays.  Re-measured on the round-2 kernels (scripts/gpu_k9ovl3.sh, profiles/r02_g/k9ovl3.txt,
// 3 reps): c3 6.98-7.05 ms sequential, 7.02-7.05 on 96 SMs, 7.06 on 112, 7.09-7.12 on 128; p124 1.94-1.95,
// 1.95-1.98, 1.98-1.99, 1.99-2.03 -- sequential stays.  RNNT_K9_CTAS=n turns the overlap on.
constexpr int kK9OverlapCtas = 0;

template <bool kPre>
__global__ void __launch_bounds__(256, 1) k7_reduce(const __nv_bfloat16* __restrict__ dx,
                                                    const __nv_bfloat16* __restrict__ h,
                                                    const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b,
                                                    int B, int Tmax, int Umax, int H, float* __restrict__ d_enc,
                                                    float* __restrict__ part) {
    __shared__ int s_part[8];
    __shared__ float4 s_enc[4][kTC][2][32];  // tree-combine slots: [slot][frame][half of the 8 columns][lane]
    const int chunk = blockIdx.x, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int off = utt_offset(T_b, U_b, b, Tmax, Umax, s_part);
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int t0 = chunk * kTC;
    const int tn = max(0, min(T - t0, kTC));
    const int c = blockIdx.z * 256 + lane * 8;
    const bool col_in = c < H;
    float enc[kTC][8];
#pragma unroll
    for (int k = 0; k < kTC; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) enc[k][e] = 0.f;
    for (int u = warp; u <= U && tn > 0 && col_in; u += 8) {
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int64_t r0 = off + static_cast<int64_t>(t0) * (U + 1) + u;
        uint4 dv[kTC], hv[kTC];
#pragma unroll
        for (int k = 0; k < kTC; ++k)  // all the unit's rows in flight before any use
            if (k < tn) {
                const int64_t r = r0 + static_cast<int64_t>(k) * (U + 1);
                dv[k] = __ldcs(reinterpret_cast<const uint4*>(dx + r * H + c));
                if (!kPre) hv[k] = __ldcs(reinterpret_cast<const uint4*>(h + r * H + c));
            }
#pragma unroll
        for (int k = 0; k < kTC; ++k)
            if (k < tn) {
                const uint32_t dw[4] = {dv[k].x, dv[k].y, dv[k].z, dv[k].w};
                uint32_t hw[4] = {0u, 0u, 0u, 0u};
                if (!kPre) hw[0] = hv[k].x, hw[1] = hv[k].y, hw[2] = hv[k].z, hw[3] = hv[k].w;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 d = unpack_bf16x2(dw[j]);
                    if (!kPre) {
                        const float2 hh = unpack_bf16x2(hw[j]);
                        d = upk(fmul2(pk(d.x, d.y), ffma2(pk(-hh.x, -hh.y), pk(hh.x, hh.y), pk(1.f, 1.f))));
                    }
                    acc[2 * j] += d.x;
                    acc[2 * j + 1] += d.y;
                    enc[k][2 * j] += d.x;
                    enc[k][2 * j + 1] += d.y;
                }
            }
        float4* pp = reinterpret_cast<float4*>(part + ((static_cast<int64_t>(chunk) * B + b) * (Umax + 1) + u) * H + c);
        pp[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        pp[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
    // tree combine of the 8 warps' d enc partials: (w, w + 4), then (w, w + 2), then (0, 1)
#pragma unroll
    for (int step = 4; step >= 1; step >>= 1) {
        if (warp >= step && warp < 2 * step) {
#pragma unroll
            for (int k = 0; k < kTC; ++k) {
                s_enc[warp - step][k][0][lane] = make_float4(enc[k][0], enc[k][1], enc[k][2], enc[k][3]);
                s_enc[warp - step][k][1][lane] = make_float4(enc[k][4], enc[k][5], enc[k][6], enc[k][7]);
            }
        }
        __syncthreads();
        if (warp < step) {
#pragma unroll
            for (int k = 0; k < kTC; ++k) {
                const float4 x = s_enc[warp][k][0][lane], y = s_enc[warp][k][1][lane];
                enc[k][0] += x.x, enc[k][1] += x.y, enc[k][2] += x.z, enc[k][3] += x.w;
                enc[k][4] += y.x, enc[k][5] += y.y, enc[k][6] += y.z, enc[k][7] += y.w;
            }
        }
        __syncthreads();
    }
    if (warp == 0 && col_in) {
#pragma unroll
        for (int k = 0; k < kTC; ++k)
            if (t0 + k < Tmax) {
                float4* o = reinterpret_cast<float4*>(d_enc + (static_cast<int64_t>(b) * Tmax + t0 + k) * H + c);
                const bool v = k < tn;
                o[0] = v ? make_float4(enc[k][0], enc[k][1], enc[k][2], enc[k][3]) : make_float4(0.f, 0.f, 0.f, 0.f);
                o[1] = v ? make_float4(enc[k][4], enc[k][5], enc[k][6], enc[k][7]) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
    }
}

// K7, pass 1, frame-per-warp form (k7_reduce_f; the default): block (chunk, b, slice) as k7_reduce, but warp w
// owns FRAME t0 + w and walks every unit: its d enc(b, t0 + w) partial is complete in 8 registers, and the 8
// warps' dpre rows of each unit are summed into the chunk's d pred partial through shared memory (groups of
// kG units: one barrier to publish, one to release; a fixed summation order: deterministic).  The next group's
// rows are loaded while the current one is combined, and ~90 registers allow 2 blocks per SM, so far more of
// each SM's bytes are in flight than with k7_reduce's 204-register warps.
// kFW warps = frames per block: 16 (512 threads, one block per SM) halves the d pred partials against 8 (two
// blocks per SM, the same 16 warps): the partials are [ceil(T / kFW)][B][U + 1][H] fp32, written here and read
// back by k7_pred_sum -- at p124 0.63 GB of traffic per step with 8-frame chunks, as much as 44 % of the dh and
// h bytes themselves.  RNNT_K7_FRAMES=8 builds the 8-frame form (A/B).
constexpr int kG = 4;
#ifndef RNNT_K7_FRAMES
#define RNNT_K7_FRAMES 16
#endif
constexpr int kFW = RNNT_K7_FRAMES;
static_assert(kFW == 8 || kFW == 16, "frames per K7 block");

constexpr size_t k7_rows_bytes() { return sizeof(float4) * kG * kFW * 2 * 32; }

template <bool kPre>
__global__ void __launch_bounds__(kFW * 32, 16 / kFW) k7_reduce_f(const __nv_bfloat16* __restrict__ dx,
                                                      const __nv_bfloat16* __restrict__ h,
                                                      const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b,
                                                      int B, int Tmax, int Umax, int H, float* __restrict__ d_enc,
                                                      float* __restrict__ part) {
    __shared__ int s_part[kFW];
    // [unit in group][warp][half of the 8 columns][lane]: 32 KB at kFW = 8, 64 KB at 16 (dynamic: > 48 KB static)
    extern __shared__ float4 k7_rows[];
    auto s_row = reinterpret_cast<float4 (*)[kFW][2][32]>(k7_rows);
    const int chunk = blockIdx.x, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int off = utt_offset(T_b, U_b, b, Tmax, Umax, s_part);
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int t0 = chunk * kFW, t = t0 + warp;
    const bool frame_in = t < T;
    const int c = blockIdx.z * 256 + lane * 8;
    const bool col_in = c < H;
    const bool ld = frame_in && col_in;
    const int64_t rbase = off + static_cast<int64_t>(t) * (U + 1);  // row of (t, u = 0)
    float enc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint4 dv[kG], hv[kG];
    auto load = [&](int u0) {
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const int u = u0 + j;
            if (ld && u <= U) {
                const int64_t r = rbase + u;
                dv[j] = __ldcs(reinterpret_cast<const uint4*>(dx + r * H + c));
                if (!kPre) hv[j] = __ldcs(reinterpret_cast<const uint4*>(h + r * H + c));
            } else {
                dv[j] = make_uint4(0u, 0u, 0u, 0u);  // bf16 zeros: contributes 0
                if (!kPre) hv[j] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
    };
    const bool any = (T > t0) && U >= 0;  // block-uniform: the chunk has frames
    if (any) load(0);
    for (int u0 = 0; any && u0 <= U; u0 += kG) {
        float d[kG][8];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const uint32_t dw[4] = {dv[j].x, dv[j].y, dv[j].z, dv[j].w};
            uint32_t hw[4] = {0u, 0u, 0u, 0u};
            if (!kPre) hw[0] = hv[j].x, hw[1] = hv[j].y, hw[2] = hv[j].z, hw[3] = hv[j].w;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 x = unpack_bf16x2(dw[e]);
                if (!kPre) {
                    const float2 hh = unpack_bf16x2(hw[e]);
                    x = upk(fmul2(pk(x.x, x.y), ffma2(pk(-hh.x, -hh.y), pk(hh.x, hh.y), pk(1.f, 1.f))));
                }
                d[j][2 * e] = x.x;
                d[j][2 * e + 1] = x.y;
                enc[2 * e] += x.x;
                enc[2 * e + 1] += x.y;
            }
        }
        if (u0 + kG <= U) load(u0 + kG);  // the next group's rows in flight while this one is combined
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            s_row[j][warp][0][lane] = make_float4(d[j][0], d[j][1], d[j][2], d[j][3]);
            s_row[j][warp][1][lane] = make_float4(d[j][4], d[j][5], d[j][6], d[j][7]);
        }
        __syncthreads();
        // thread of warps 0-7 -> (unit j = warp / 2, half = warp & 1, lane): sums the kFW frames' rows in warp order
        if (warp < 2 * kG) {
            const int j = warp >> 1, hf = warp & 1;
            const int u = u0 + j;
            if (u <= U && col_in) {
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < kFW; ++w) {
                    const float4 x = s_row[j][w][hf][lane];
                    o.x += x.x, o.y += x.y, o.z += x.z, o.w += x.w;
                }
                reinterpret_cast<float4*>(part + ((static_cast<int64_t>(chunk) * B + b) * (Umax + 1) + u) * H + c)[hf] = o;
            }
        }
        __syncthreads();
    }
    if (col_in && t < Tmax) {
        float4* o = reinterpret_cast<float4*>(d_enc + (static_cast<int64_t>(b) * Tmax + t) * H + c);
        o[0] = frame_in ? make_float4(enc[0], enc[1], enc[2], enc[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
        o[1] = frame_in ? make_float4(enc[4], enc[5], enc[6], enc[7]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// K7, pass 2: d pred(b, u, :) = sum over the chunks covering frames < T_b of pass 1's partials (chunk order);
// padded units (and invalid utterances) get 0.  Block (u, b), 128 threads x 4 columns.
__global__ void __launch_bounds__(128) k7_pred_sum(const float* __restrict__ part, const int32_t* __restrict__ T_b,
                                                   const int32_t* __restrict__ U_b, int B, int Tmax, int Umax, int H,
                                                   int tc, float* __restrict__ d_pred) {  // tc: frames per chunk
    const int u = blockIdx.x, b = blockIdx.y;
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int nch = (u <= U) ? (T + tc - 1) / tc : 0;
    for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
        // chunk order kept (deterministic); eight loads in flight before their adds (a chain of dependent global
        // loads otherwise)
        auto at = [&](int ch) {
            return __ldcs(reinterpret_cast<const float4*>(part + ((static_cast<int64_t>(ch) * B + b) * (Umax + 1) + u) * H + c));
        };
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        int ch = 0;
        for (; ch + 8 <= nch; ch += 8) {
            float4 p[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) p[k] = at(ch + k);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                o.x += p[k].x;
                o.y += p[k].y;
                o.z += p[k].z;
                o.w += p[k].w;
            }
        }
        for (; ch < nch; ++ch) {
            const float4 p = at(ch);
            o.x += p.x;
            o.y += p.y;
            o.z += p.z;
            o.w += p.w;
        }
        *reinterpret_cast<float4*>(d_pred + (static_cast<int64_t>(b) * (Umax + 1) + u) * H + c) = o;
    }
}

struct GradLayout {
    int64_t R;  // padded rows B * Tmax * (Umax + 1)
    int Vp;
    size_t base, rowmap, nrows, dz, h, dpre, part, kpart, total;
};

GradLayout grad_layout(int B, int Tmax, int Umax, int H, int V) {
    GradLayout L{};
    L.R = static_cast<int64_t>(B) * Tmax * (Umax + 1);
    L.Vp = (V + kJointVTile - 1) / kJointVTile * kJointVTile;
    size_t off = align256(workspace_bytes(B, Tmax, Umax));
    L.base = 0;
    L.rowmap = off;
    off += align256(sizeof(int) * L.R);
    L.nrows = off;
    off += 256;
    L.dz = off;
    off += align256(sizeof(__nv_bfloat16) * L.R * L.Vp);
    L.h = off;
    off += align256(sizeof(__nv_bfloat16) * L.R * H);
    L.dpre = off;  // K8's output [R][H] bf16: dh (or dpre)
    off += align256(sizeof(__nv_bfloat16) * L.R * H);
    L.part = off;  // K9's per-row-range partials of dW and dbias
    off += align256(k9_partial_bytes(L.Vp, H));
    L.kpart = off;  // K7's per-frame-chunk partials of d pred [ceil(Tmax / tc)][B][Umax + 1][H] fp32, tc >= kTC
    off += align256(sizeof(float) * static_cast<size_t>((Tmax + kTC - 1) / kTC) * B * (Umax + 1) * H);
    L.total = off;
    return L;
}

}  // namespace
}  // namespace rnnt

extern "C" size_t rnnt_joint_grad_workspace_bytes(int B, int Tmax, int Umax, int H, int V) {
    if (B < 0 || Tmax < 1 || Umax < 0 || H < 1 || V < 2) return 0;
    return rnnt::grad_layout(B, Tmax, Umax, H, V).total;
}

extern "C" rnnt_status rnnt_joint_loss_grad(const void* enc, const void* pred, const void* weight, const float* bias,
                                            const int32_t* targets, const int32_t* logit_lens,
                                            const int32_t* target_lens, int B, int Tmax, int Umax, int H, int V,
                                            int blank, int variant, float* losses, float* d_enc, float* d_pred,
                                            float* d_weight, float* d_bias, const float* grad_scale,
                                            int64_t valid_rows, void* workspace, size_t workspace_bytes,
                                            void* stream) {
    using namespace rnnt;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (B < 0 || Tmax < 1 || Umax < 0 || H < 1 || V < 2) return RNNT_ERR_INVALID_ARG;
    if (B == 0) return RNNT_OK;
    if (!losses || !d_enc || !d_pred || !d_weight || !workspace) return RNNT_ERR_INVALID_ARG;
    const GradLayout L = grad_layout(B, Tmax, Umax, H, V);
    if (workspace_bytes < L.total) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    if (L.R >= (int64_t(1) << 31)) return RNNT_ERR_UNSUPPORTED;
    if (valid_rows < -1 || valid_rows > L.R) return RNNT_ERR_INVALID_ARG;
    char* ws = static_cast<char*>(workspace);
    int* rowmap = reinterpret_cast<int*>(ws + L.rowmap);
    int* nrows = reinterpret_cast<int*>(ws + L.nrows);
    auto* dz = reinterpret_cast<__nv_bfloat16*>(ws + L.dz);
    auto* hb = reinterpret_cast<__nv_bfloat16*>(ws + L.h);
    auto* dpre = reinterpret_cast<__nv_bfloat16*>(ws + L.dpre);
    auto* part = reinterpret_cast<float*>(ws + L.part);
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    // forward: K6 (row map into the gradient workspace, which K2 does not touch) and K2 (alpha, beta, losses)
    // The forward also stores h (from its builders' registers) so that K6<grad> loads it by TMA instead of
    // recomputing tanh(f + g) (RNNT_K6_HREUSE=0: K6<grad> recomputes and stores h, for A/B).
    const bool hreuse = !(getenv("RNNT_K6_HREUSE") && atoi(getenv("RNNT_K6_HREUSE")) == 0);
    rnnt_status st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V,
                                 blank, workspace, workspace_bytes, s, nullptr, rowmap, nrows, true, nullptr,
                                 hreuse ? hb : nullptr);
    if (st != RNNT_OK) return st;
    const Workspace w = carve(workspace, B, Tmax, Umax);
    const int vk = (variant < 0) ? kRnnt : (variant == WRNNT_FORCE_FINAL ? kForceFinal : kAllowIgnore);
    Problem p{nullptr, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, vk, losses, nullptr, nullptr, kF32};
    if (launch_k2_alpha_beta(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
    // backward pass 1: z again on the tensor cores -> dz (bf16) (and h when the forward did not store it)
    const GradIO g{w.lse, w.lp, w.alpha, w.beta, w.logp, grad_scale, dz, hb, hreuse};
    st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V, blank,
                     workspace, workspace_bytes, s, nullptr, rowmap, nrows, false, &g);
    if (st != RNNT_OK) return st;
    // rows the GEMMs cover: the caller's valid-row count (no padded rows: no zeroing, no wasted GEMM work), else
    // every padded row with the tail [*nrows, R) zeroed on the device
    const int R = static_cast<int>(valid_rows >= 0 ? valid_rows : L.R);
    if (valid_rows < 0) {
        k7_zero_tail<<<1184, 256, 0, s>>>(nrows, L.R, L.Vp, H, dz, hb);
    } else {
        k7_check_rows<<<1, 256, 0, s>>>(nrows, valid_rows, B, losses);
    }
    if (cudaGetLastError() != cudaSuccess) return RNNT_ERR_CUDA;
    // K8: dh = dz W (bf16; RNNT_K8_TANH=1: dpre = dh * (1 - h^2) in K8's epilogue, A/B), on every SM.  Then K9
    // (dW, dbias: tensor-bound) and K7 (tanh' + reductions: HBM-bound) run side by side: K9 on an internal
    // high-priority stream with its grid capped at kK9OverlapCtas SMs, K7 on the caller's stream filling the
    // SMs K9 leaves (neither fits on an SM next to the other: K9 holds ~200 KB of shared memory); the caller's
    // stream then joins K9 back.  RNNT_K9_CTAS=n sets the cap (0: K9 on every SM, then K7: sequential).
    const bool tanh_k8 = getenv("RNNT_K8_TANH") && atoi(getenv("RNNT_K8_TANH")) != 0;
    if (launch_k8(dz, static_cast<const __nv_bfloat16*>(weight), hb, dpre, R, H, H, V, L.Vp, tanh_k8, s) != cudaSuccess)
        return RNNT_ERR_CUDA;
    int k9_ctas = kK9OverlapCtas;
    if (const char* e = getenv("RNNT_K9_CTAS")) k9_ctas = atoi(e);
    AuxPool* pool = k9_ctas > 0 ? aux_pool() : nullptr;
    cudaStream_t k9s = s;
    if (pool) {
        k9s = pool->aux[0];
        if (cudaEventRecord(pool->k1_done[0], s) != cudaSuccess || cudaStreamWaitEvent(k9s, pool->k1_done[0], 0) != cudaSuccess)
            return RNNT_ERR_CUDA;
    }
    if (launch_k9(dz, hb, R, H, H, V, L.Vp, part, d_weight, d_bias, k9s, pool ? k9_ctas : 0) != cudaSuccess)
        return RNNT_ERR_CUDA;
    if (pool && cudaEventRecord(pool->k2_done[0], k9s) != cudaSuccess) return RNNT_ERR_CUDA;
    // K7: tanh' and the reductions into d enc / d pred (its d pred partials in their own region: K9 may still
    // be reading dz)
    float* ppart = reinterpret_cast<float*>(ws + L.kpart);
    const bool k7_units = getenv("RNNT_K7_UNITS") && atoi(getenv("RNNT_K7_UNITS")) != 0;  // A/B: unit-per-warp K7
    const int tc = k7_units ? kTC : kFW;  // frames per d pred partial
    // k7_reduce_f's dynamic shared memory above the 48 KB default (set per call: the attribute is per device)
    if (!k7_units && cudaFuncSetAttribute(tanh_k8 ? k7_reduce_f<true> : k7_reduce_f<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(k7_rows_bytes())) != cudaSuccess)
        return RNNT_ERR_CUDA;
    const dim3 g7((Tmax + tc - 1) / tc, B, (H + 255) / 256);
    if (k7_units) {
        if (tanh_k8)
            k7_reduce<true><<<g7, 256, 0, s>>>(dpre, nullptr, logit_lens, target_lens, B, Tmax, Umax, H, d_enc, ppart);
        else
            k7_reduce<false><<<g7, 256, 0, s>>>(dpre, hb, logit_lens, target_lens, B, Tmax, Umax, H, d_enc, ppart);
    } else {
        if (tanh_k8)
            k7_reduce_f<true><<<g7, kFW * 32, k7_rows_bytes(), s>>>(dpre, nullptr, logit_lens, target_lens, B, Tmax, Umax,
                                                                      H, d_enc, ppart);
        else
            k7_reduce_f<false><<<g7, kFW * 32, k7_rows_bytes(), s>>>(dpre, hb, logit_lens, target_lens, B, Tmax, Umax, H,
                                                                       d_enc, ppart);
    }
    k7_pred_sum<<<dim3(Umax + 1, B), 128, 0, s>>>(ppart, logit_lens, target_lens, B, Tmax, Umax, H, tc, d_pred);
    if (cudaGetLastError() != cudaSuccess) return RNNT_ERR_CUDA;
    if (pool && cudaStreamWaitEvent(s, pool->k2_done[0], 0) != cudaSuccess) return RNNT_ERR_CUDA;  // join K9
    return RNNT_OK;
}
