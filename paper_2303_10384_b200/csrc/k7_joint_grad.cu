// k7_joint_grad.cu -- the backward of the fused joint network + loss (training).
//
// Gradients of sum_b loss_b with respect to the joint's inputs (readings R22, R23):
//   dz(t,u,v)  = softmax(z)(v) (occ_b + occ_y) - [v = blank] occ_b - [v = y_u] occ_y      (K3's formula)
//   dh(t,u,:)  = sum_v dz(t,u,v) W(v,:)                  dW(v,:) = sum_{t,u} dz(t,u,v) h(t,u,:)
//   dbias(v)   = sum_{t,u} dz(t,u,v)
//   dpre       = dh * (1 - h^2)   (dh stored in bf16, tanh' from the stored bf16 h)
//   d enc(b,t,:) = sum_{u <= U_b} dpre(t,u,:)           d pred(b,u,:) = sum_{t < T_b} dpre(t,u,:)
// over the valid cells.  Pipeline (all on the caller's stream):
//   K6 (forward: lse, gathers) -> K2 (alpha, beta, losses) -> K6<grad> (recomputes z on the tensor cores;
//   its epilogue writes dz in bf16, its builders write h with an extra (1, 0, .., 0) column) -> two plain
//   cuBLAS GEMMs (dh = dz W; [dW | dbias] = dz^T [h | 1], bf16 in, fp32 accumulate and out) -> K7 (tanh' and
//   the two reductions).  The [B,T,U+1,V] logits never exist; dz does, in bf16 (half the bytes of fp32 logits),
//   because dW needs it against every row.  Rows are the compact valid cells (K6's row map); the GEMMs run
//   over the padded row count B*Tmax*(Umax+1) (the host does not know the valid count without a sync) with
//   the tail rows zeroed.
#include <algorithm>

#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "elem.cuh"
#include "joint.cuh"
#include "rnnt_b200.h"

namespace rnnt {
namespace {

constexpr int kJointMaxDevices = 64;

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

// W [V][H] -> Wp [Vp][H], rows V..Vp-1 zero (dz's tail columns are zero too: K = Vp adds nothing).
__global__ void __launch_bounds__(256) k7_pad_w(const __nv_bfloat16* __restrict__ w, int V, int Vp, int H,
                                                __nv_bfloat16* __restrict__ wp) {
    const int64_t n = static_cast<int64_t>(Vp) * H / 8, nv = static_cast<int64_t>(V) * H / 8;  // 16-byte units
    const uint4* w4 = reinterpret_cast<const uint4*>(w);
    uint4* o4 = reinterpret_cast<uint4*>(wp);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        o4[i] = i < nv ? w4[i] : make_uint4(0u, 0u, 0u, 0u);
}

// valid_rows given by the caller must equal the row map's count; else every loss is NaN (loud failure: the
// GEMMs ran over the wrong rows).
__global__ void k7_check_rows(const int* __restrict__ nrows, int64_t valid_rows, int B, float* __restrict__ losses) {
    if (*nrows == valid_rows) return;
    for (int i = threadIdx.x; i < B; i += blockDim.x) losses[i] = __int_as_float(0x7fc00000);
}

// d_weight [V][H] and d_bias [V] out of the augmented dW GEMM's [V][H + kJointHPad] result.
__global__ void __launch_bounds__(256) k7_split_dw(const float* __restrict__ dwa, int V, int H, float* __restrict__ dw,
                                                   float* __restrict__ db) {
    const int Hs = H + kJointHPad;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < static_cast<int64_t>(V) * Hs;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int v = static_cast<int>(i / Hs), c = static_cast<int>(i - static_cast<int64_t>(v) * Hs);
        if (c < H)
            dw[static_cast<int64_t>(v) * H + c] = dwa[i];
        else if (c == H && db)
            db[v] = dwa[i];
    }
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

// K7, pass 1: block (chunk, b, slice) takes frames [chunk * kTC, +kTC) of utterance b and a 128-column slice
// of H, and reads each of its rows of dh and h ONCE: dpre = dh * (1 - h^2).  Warp w owns units u = w (mod 4):
// its sum over the chunk's frames is the chunk's partial of d pred(b, u) (-> part, registers); its
// contribution to d enc(b, t) is added to a per-warp shared-memory partial, summed over the four warps in a
// fixed order at the end (the block owns every unit of its frames: d enc is complete, written directly).
// Pass 2 sums the chunk partials of d pred in chunk order.  Deterministic; 128 threads x 4 columns.
// (Replaces one pass per output, which read dh and h twice: 1.19 -> 0.81 ms at c3, ncu launch list.)
constexpr int kTC = 8;

__global__ void __launch_bounds__(128) k7_reduce(const __nv_bfloat16* __restrict__ dh, const __nv_bfloat16* __restrict__ h,
                                                 const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b,
                                                 int B, int Tmax, int Umax, int H, float* __restrict__ d_enc,
                                                 float* __restrict__ part) {
    __shared__ int s_part[4];
    __shared__ float4 s_enc[4][kTC][32];
    const int chunk = blockIdx.x, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int off = utt_offset(T_b, U_b, b, Tmax, Umax, s_part);
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int t0 = chunk * kTC;
    const int tn = max(0, min(T - t0, kTC));
    const int c = blockIdx.z * 128 + lane * 4;
    const int Hg = H + kJointHGPad;
    float4 enc[kTC];  // this warp's partial of d enc(b, t0 + k) over its units (registers; shared at the end)
#pragma unroll
    for (int k = 0; k < kTC; ++k) enc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int u = warp; u <= U && tn > 0; u += 4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t r0 = off + static_cast<int64_t>(t0) * (U + 1) + u;
        auto row = [&](int k, uint2 dw, uint2 hw) {
            const float h0 = __uint_as_float(hw.x << 16), h1 = __uint_as_float(hw.x & 0xffff0000u);
            const float h2 = __uint_as_float(hw.y << 16), h3 = __uint_as_float(hw.y & 0xffff0000u);
            float4 d;
            d.x = __uint_as_float(dw.x << 16) * fmaf(-h0, h0, 1.f);
            d.y = __uint_as_float(dw.x & 0xffff0000u) * fmaf(-h1, h1, 1.f);
            d.z = __uint_as_float(dw.y << 16) * fmaf(-h2, h2, 1.f);
            d.w = __uint_as_float(dw.y & 0xffff0000u) * fmaf(-h3, h3, 1.f);
            acc.x += d.x;
            acc.y += d.y;
            acc.z += d.z;
            acc.w += d.w;
            float4& e = enc[k];
            e.x += d.x;
            e.y += d.y;
            e.z += d.z;
            e.w += d.w;
        };
        auto ld = [&](int k, uint2& dw, uint2& hw) {
            const int64_t r = r0 + static_cast<int64_t>(k) * (U + 1);
            dw = __ldcs(reinterpret_cast<const uint2*>(dh + r * H + c));
            hw = __ldcs(reinterpret_cast<const uint2*>(h + r * Hg + c));
        };
        if (tn == kTC) {  // whole chunk: all kTC rows' loads issued before any use
            uint2 dw[kTC], hw[kTC];
#pragma unroll
            for (int k = 0; k < kTC; ++k) ld(k, dw[k], hw[k]);
#pragma unroll
            for (int k = 0; k < kTC; ++k) row(k, dw[k], hw[k]);
        } else {
#pragma unroll
            for (int k = 0; k < kTC; ++k)  // unrolled so enc[] stays in registers
                if (k < tn) {
                    uint2 dw, hw;
                    ld(k, dw, hw);
                    row(k, dw, hw);
                }
        }
        *reinterpret_cast<float4*>(part + ((static_cast<int64_t>(chunk) * B + b) * (Umax + 1) + u) * H + c) = acc;
    }
#pragma unroll
    for (int k = 0; k < kTC; ++k) s_enc[warp][k][lane] = enc[k];
    __syncthreads();
    for (int k = warp; k < kTC && t0 + k < Tmax; k += 4) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < tn) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float4 e = s_enc[w][k][lane];
                o.x += e.x;
                o.y += e.y;
                o.z += e.z;
                o.w += e.w;
            }
        }
        *reinterpret_cast<float4*>(d_enc + (static_cast<int64_t>(b) * Tmax + t0 + k) * H + c) = o;
    }
}

// K7, pass 2: d pred(b, u, :) = sum over the chunks covering frames < T_b of pass 1's partials (chunk order);
// padded units (and invalid utterances) get 0.  Block (u, b), 128 threads x 4 columns.
__global__ void __launch_bounds__(128) k7_pred_sum(const float* __restrict__ part, const int32_t* __restrict__ T_b,
                                                   const int32_t* __restrict__ U_b, int B, int Tmax, int Umax, int H,
                                                   float* __restrict__ d_pred) {
    const int u = blockIdx.x, b = blockIdx.y;
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int nch = (u <= U) ? (T + kTC - 1) / kTC : 0;
    for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int ch = 0; ch < nch; ++ch) {
            const float4 p = __ldcs(reinterpret_cast<const float4*>(part + ((static_cast<int64_t>(ch) * B + b) * (Umax + 1) + u) * H + c));
            o.x += p.x;
            o.y += p.y;
            o.z += p.z;
            o.w += p.w;
        }
        *reinterpret_cast<float4*>(d_pred + (static_cast<int64_t>(b) * (Umax + 1) + u) * H + c) = o;
    }
}

// Per host thread and device: one cuBLAS handle (creating one per call costs milliseconds).
cublasHandle_t blas_handle() {
    thread_local cublasHandle_t handles[kJointMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kJointMaxDevices) return nullptr;
    if (!handles[dev] && cublasCreate(&handles[dev]) != CUBLAS_STATUS_SUCCESS) handles[dev] = nullptr;
    return handles[dev];
}

struct GradLayout {
    int64_t R;  // padded rows B * Tmax * (Umax + 1)
    int Vp;
    size_t base, rowmap, nrows, dz, h, dh, dwa, wp, total;
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
    L.dz = off;  // dz; after the two GEMMs, K7's d pred partials [ceil(Tmax / kTC)][B][Umax + 1][H] fp32
    off += align256(std::max(sizeof(__nv_bfloat16) * L.R * L.Vp,
                             sizeof(float) * static_cast<size_t>((Tmax + kTC - 1) / kTC) * B * (Umax + 1) * H));
    L.h = off;
    off += align256(sizeof(__nv_bfloat16) * L.R * (H + kJointHGPad));
    L.dh = off;
    off += align256(sizeof(__nv_bfloat16) * L.R * H);
    L.dwa = off;
    off += align256(sizeof(float) * static_cast<size_t>(V) * (H + kJointHPad));
    L.wp = off;  // W padded to Vp rows (zero tail) when V % kJointVTile != 0: the dh GEMM runs with K = Vp
    off += align256(sizeof(__nv_bfloat16) * static_cast<size_t>(L.Vp) * H);
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
    auto* dh = reinterpret_cast<__nv_bfloat16*>(ws + L.dh);
    auto* dwa = reinterpret_cast<float*>(ws + L.dwa);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cublasHandle_t hd = blas_handle();
    if (!hd) return RNNT_ERR_CUDA;

    // forward: K6 (row map into the gradient workspace, which K2 does not touch) and K2 (alpha, beta, losses)
    rnnt_status st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V,
                                 blank, workspace, workspace_bytes, s, nullptr, rowmap, nrows, true, nullptr);
    if (st != RNNT_OK) return st;
    const Workspace w = carve(workspace, B, Tmax, Umax);
    const int vk = (variant < 0) ? kRnnt : (variant == WRNNT_FORCE_FINAL ? kForceFinal : kAllowIgnore);
    Problem p{nullptr, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, vk, losses, nullptr, nullptr, kF32};
    if (launch_k2_alpha_beta(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
    // backward pass 1: z again on the tensor cores -> dz (bf16), h
    const GradIO g{w.lse, w.lp, w.alpha, w.beta, w.logp, grad_scale, dz, hb};
    st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V, blank,
                     workspace, workspace_bytes, s, nullptr, rowmap, nrows, false, &g);
    if (st != RNNT_OK) return st;
    const int Hs = H + kJointHPad;
    // rows the GEMMs cover: the caller's valid-row count (no padded rows: no zeroing, no wasted GEMM work), else
    // every padded row with the tail [*nrows, R) zeroed on the device
    const int R = static_cast<int>(valid_rows >= 0 ? valid_rows : L.R);
    if (valid_rows < 0) {
        k7_zero_tail<<<1184, 256, 0, s>>>(nrows, L.R, L.Vp, H + kJointHGPad, dz, hb);
    } else {
        k7_check_rows<<<1, 256, 0, s>>>(nrows, valid_rows, B, losses);
    }
    if (cudaGetLastError() != cudaSuccess) return RNNT_ERR_CUDA;
    const void* wk = weight;  // dh GEMM's W: K = Vp (a multiple of the tile) keeps cuBLAS on its sm_100 kernels
    if (L.Vp != V) {
        auto* wp = reinterpret_cast<__nv_bfloat16*>(ws + L.wp);
        k7_pad_w<<<148, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(weight), V, L.Vp, H, wp);
        if (cudaGetLastError() != cudaSuccess) return RNNT_ERR_CUDA;
        wk = wp;
    }
    // the two GEMMs and dbias (column-major views of the row-major arrays; bf16 in, fp32 accumulate / out)
    const float one = 1.f, zero = 0.f;
    if (cublasSetStream(hd, s) != CUBLAS_STATUS_SUCCESS) return RNNT_ERR_CUDA;
    if (R == 0) {
        if (cudaMemsetAsync(dwa, 0, sizeof(float) * static_cast<size_t>(V) * Hs, s) != cudaSuccess) return RNNT_ERR_CUDA;
    } else {
        // dh^T [H x R] = W^T [H x Vp] . dz^T [Vp x R]
        if (cublasGemmEx(hd, CUBLAS_OP_N, CUBLAS_OP_N, H, R, L.Vp, &one, wk, CUDA_R_16BF, H, dz, CUDA_R_16BF, L.Vp,
                         &zero, dh, CUDA_R_16BF, H, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
            return RNNT_ERR_CUDA;
        // [dW | dbias]^T [(H + 8) x V] = [h | 1 0..0]^T [(H + 8) x R] . dz [R x V]
        if (cublasGemmEx(hd, CUBLAS_OP_N, CUBLAS_OP_T, Hs, V, R, &one, hb, CUDA_R_16BF, H + kJointHGPad, dz, CUDA_R_16BF, L.Vp,
                         &zero, dwa, CUDA_R_32F, Hs, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
            return RNNT_ERR_CUDA;
    }
    k7_split_dw<<<296, 256, 0, s>>>(dwa, V, H, d_weight, d_bias);
    // K7: tanh' and the reductions into d enc / d pred
    float* part = reinterpret_cast<float*>(ws + L.dz);  // dz is dead after the GEMMs
    k7_reduce<<<dim3((Tmax + kTC - 1) / kTC, B, H / 128), 128, 0, s>>>(dh, hb, logit_lens, target_lens, B, Tmax, Umax,
                                                                       H, d_enc, part);
    k7_pred_sum<<<dim3(Umax + 1, B), 128, 0, s>>>(part, logit_lens, target_lens, B, Tmax, Umax, H, d_pred);
    return cudaGetLastError() == cudaSuccess ? RNNT_OK : RNNT_ERR_CUDA;
}
