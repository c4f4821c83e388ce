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

// Zero rows [*nrows, R) of dz ([R][Vp]) and h ([R][Hs]) so the padded-row GEMMs see no stale data.
__global__ void __launch_bounds__(256) k7_zero_tail(const int* __restrict__ nrows, int64_t R, int Vp, int Hs,
                                                    __nv_bfloat16* dz, __nv_bfloat16* h) {
    const int64_t r0 = *nrows;
    const int64_t nz = (R - r0) * Vp / 8, nh = (R - r0) * Hs / 8;  // 16-byte units
    uint4* z4 = reinterpret_cast<uint4*>(dz + r0 * Vp);
    uint4* h4 = reinterpret_cast<uint4*>(h + r0 * Hs);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nz + nh;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < nz)
            z4[i] = make_uint4(0u, 0u, 0u, 0u);
        else
            h4[i - nz] = make_uint4(0u, 0u, 0u, 0u);
    }
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

// K7: block (i, b) reduces dpre = dh * (1 - h^2) over u for frame i (mode 0: d enc[b, i, :]) or over t for
// unit i (mode 1: d pred[b, i, :]); H <= 512, 128 threads x 4 columns; padded frames / units get 0.  (One
// pass computing both with shared-memory partials and atomics measured slower: 2.5 vs 1.4 ms at c3.)
template <int kMode>
__global__ void __launch_bounds__(128) k7_reduce(const __nv_bfloat16* __restrict__ dh, const __nv_bfloat16* __restrict__ h,
                                                 const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b,
                                                 int Tmax, int Umax, int H, float* __restrict__ out) {
    __shared__ int s_part[4];
    const int i = blockIdx.x, b = blockIdx.y;
    const int off = utt_offset(T_b, U_b, b, Tmax, Umax, s_part);
    const int n = utt_count(T_b, U_b, b, Tmax, Umax);
    const int T = n ? T_b[b] : 0, U = n ? U_b[b] : -1;
    const int len = kMode == 0 ? (i < T ? U + 1 : 0) : (i <= U ? T : 0);
    const int64_t first = off + (kMode == 0 ? static_cast<int64_t>(i) * (U + 1) : i);
    const int64_t stride = kMode == 0 ? 1 : (U + 1);
    const int Hs = H + kJointHPad;
    float* o = out + (static_cast<int64_t>(b) * (kMode == 0 ? Tmax : Umax + 1) + i) * H;
    for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int k = 0; k < len; ++k) {
            const int64_t r = first + k * stride;
            const uint2 dw = *reinterpret_cast<const uint2*>(dh + r * H + c);
            const float4 d = make_float4(__uint_as_float(dw.x << 16), __uint_as_float(dw.x & 0xffff0000u),
                                         __uint_as_float(dw.y << 16), __uint_as_float(dw.y & 0xffff0000u));
            const uint2 hw = *reinterpret_cast<const uint2*>(h + r * Hs + c);
            const float h0 = __uint_as_float(hw.x << 16), h1 = __uint_as_float(hw.x & 0xffff0000u);
            const float h2 = __uint_as_float(hw.y << 16), h3 = __uint_as_float(hw.y & 0xffff0000u);
            acc.x = fmaf(d.x, fmaf(-h0, h0, 1.f), acc.x);
            acc.y = fmaf(d.y, fmaf(-h1, h1, 1.f), acc.y);
            acc.z = fmaf(d.z, fmaf(-h2, h2, 1.f), acc.z);
            acc.w = fmaf(d.w, fmaf(-h3, h3, 1.f), acc.w);
        }
        *reinterpret_cast<float4*>(o + c) = acc;
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
    size_t base, rowmap, nrows, dz, h, dh, dwa, total;
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
    off += align256(sizeof(__nv_bfloat16) * L.R * (H + kJointHPad));
    L.dh = off;
    off += align256(sizeof(__nv_bfloat16) * L.R * H);
    L.dwa = off;
    off += align256(sizeof(float) * static_cast<size_t>(V) * (H + kJointHPad));
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
                                            void* workspace, size_t workspace_bytes, void* stream) {
    using namespace rnnt;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (B < 0 || Tmax < 1 || Umax < 0 || H < 1 || V < 2) return RNNT_ERR_INVALID_ARG;
    if (B == 0) return RNNT_OK;
    if (!losses || !d_enc || !d_pred || !d_weight || !workspace) return RNNT_ERR_INVALID_ARG;
    const GradLayout L = grad_layout(B, Tmax, Umax, H, V);
    if (workspace_bytes < L.total) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    if (L.R >= (int64_t(1) << 31)) return RNNT_ERR_UNSUPPORTED;
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
    k7_zero_tail<<<1184, 256, 0, s>>>(nrows, L.R, L.Vp, Hs, dz, hb);
    if (cudaGetLastError() != cudaSuccess) return RNNT_ERR_CUDA;
    // the two GEMMs and dbias (column-major views of the row-major arrays; bf16 in, fp32 accumulate / out)
    const float one = 1.f, zero = 0.f;
    const int R = static_cast<int>(L.R);
    if (cublasSetStream(hd, s) != CUBLAS_STATUS_SUCCESS) return RNNT_ERR_CUDA;
    // dh^T [H x R] = W^T [H x V] . dz^T [V x R]
    if (cublasGemmEx(hd, CUBLAS_OP_N, CUBLAS_OP_N, H, R, V, &one, weight, CUDA_R_16BF, H, dz, CUDA_R_16BF, L.Vp,
                     &zero, dh, CUDA_R_16BF, H, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
        return RNNT_ERR_CUDA;
    // [dW | dbias]^T [(H + 8) x V] = [h | 1 0..0]^T [(H + 8) x R] . dz [R x V]
    if (cublasGemmEx(hd, CUBLAS_OP_N, CUBLAS_OP_T, Hs, V, R, &one, hb, CUDA_R_16BF, Hs, dz, CUDA_R_16BF, L.Vp, &zero,
                     dwa, CUDA_R_32F, Hs, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
        return RNNT_ERR_CUDA;
    k7_split_dw<<<296, 256, 0, s>>>(dwa, V, H, d_weight, d_bias);
    // K7: tanh' and the reductions into d enc / d pred
    k7_reduce<0><<<dim3(Tmax, B), 128, 0, s>>>(dh, hb, logit_lens, target_lens, Tmax, Umax, H, d_enc);
    k7_reduce<1><<<dim3(Umax + 1, B), 128, 0, s>>>(dh, hb, logit_lens, target_lens, Tmax, Umax, H, d_pred);
    return cudaGetLastError() == cudaSuccess ? RNNT_OK : RNNT_ERR_CUDA;
}
