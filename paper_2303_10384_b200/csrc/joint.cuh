// joint.cuh -- internal interface between the fused joint's forward / first backward pass (k6_joint.cu) and
// the rest of its backward (k7_joint_grad.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rnnt_b200.h"

namespace rnnt {

// Backward-pass inputs / outputs of K6<true>: the forward's lse / lp and K2's alpha / beta / logP in; dz
// ([rows][Vp] bf16, Vp = V rounded up to 128) and h ([rows][H] bf16) out, rows = the compact valid cells.
struct GradIO {
    const float* lse;
    const double2* lp;
    const double* alpha;
    const double* beta;
    const double* logp;
    const float* grad_scale;  // [B] or nullptr (= 1): dz of utterance b is scaled by it (e.g. 1/B for a mean)
    __nv_bfloat16* dz;
    __nv_bfloat16* h;
    bool h_ready;  // h already holds the rows (the forward stored them, joint_front's h_fwd): K6 loads h
                   // instead of recomputing tanh(f + g); else K6 computes and stores it
};

// Argument checks, W's tensor map, (optionally) the compact row map, and K6: the forward (-> lse and the
// Populate gathers in the workspace) when g == nullptr, the backward's first pass (-> dz, h) otherwise.
// rowmap / nrows: where the row map lives (nullptr: the workspace's alpha / beta regions, free until K2).
// h_fwd (forward only): the builders also store h = bf16(tanh(f + g)) there ([rows][H], compact rows), for a
// later K6<grad> with GradIO::h_ready.
rnnt_status joint_front(const void* enc, const void* pred, const void* weight, const float* bias,
                        const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens, int B,
                        int Tmax, int Umax, int H, int V, int blank, void* workspace, size_t workspace_bytes,
                        cudaStream_t s, void* const* events, int* rowmap = nullptr, int* nrows = nullptr,
                        bool make_map = true, const GradIO* g = nullptr, __nv_bfloat16* h_fwd = nullptr);

// K8 / K9 (k8_joint_bwd.cu): the backward GEMMs on the tensor cores.  K8: out = bf16(dz W) over R rows, or with
// tanh_in_k8 bf16((dz W) * (1 - h^2)) (the pair kernel; the 2-D cluster A/B kernel always applies it); K9:
// d_weight = dz^T h, d_bias = column sums of dz (d_bias may be nullptr), through `part` (k9_partial_bytes).
// dz [R][Vp], h [R][Hg] (row pitch Hg), W [V][H], out [R][H]; H % 128 == 0, H <= 512.
size_t k9_partial_bytes(int Vp, int H);
cudaError_t launch_k8(const __nv_bfloat16* dz, const __nv_bfloat16* weight, const __nv_bfloat16* h,
                      __nv_bfloat16* out, int R, int H, int Hg, int V, int Vp, bool tanh_in_k8, cudaStream_t s);
// max_ctas > 0 caps K9's grid (the rest of the SMs run K7 concurrently); 0 = every co-resident pair.
cudaError_t launch_k9(const __nv_bfloat16* dz, const __nv_bfloat16* h, int R, int H, int Hg, int V, int Vp,
                      float* part, float* d_weight, float* d_bias, cudaStream_t s, int max_ctas = 0);

constexpr int kJointVTile = 128;  // K6's N tile: dz rows are padded to a multiple of it
constexpr int kJointHPad = 8;     // K6's A staging rows: H + 8 bf16 (16 bytes of pad: conflict-free row reads)
// h's global row stride beyond H: none (rows of H bf16 = 256 .. 1024 bytes, 128-byte aligned); round 1 carried a
// (1, 0, .., 0) column for a library dbias GEMM and a 128-byte aligned stride H + 64 for K7.
constexpr int kJointHGPad = 0;

}  // namespace rnnt
