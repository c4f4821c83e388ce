// k6_joint.cu -- K6: the joint network fused with K1: the logits tensor is never
// materialised.
//
// PAPER.md §4.1: the benchmark pipeline feeds the loss from a joint network over Encoder and Predictor
// embeddings of size 512; the log-probabilities tensor X comes from that network.  The joint here
// is the standard transducer joiner (reading R22):
//   h(b,t,u,:) = bf16( tanh( f(b,t,:) + g(b,u,:) ) )            f: [B,Tmax,H], g: [B,Umax+1,H] bf16
//   z(b,t,u,v) = sum_k h(b,t,u,k) W(v,k) + bias(v)                W: [V,H] bf16, bias fp32, fp32 accumulate
// and K6 produces exactly what K1 produces from z -- lse(t,u) and the Populate gathers X_b, X_y (§2.2 Eq.(3)
// P:88) in K2's anti-diagonal layout -- so K2 then yields the losses unchanged.
//
// One persistent CTA per SM (20 warps), rows = the valid (b,t,u) cells (k6_rowmap) in tiles of 128:
//   warp 0       TMA producer: W tiles [128 v x 64 k] (SWIZZLE_128B) into a ring of kStages smem stages
//   warp 1       TMEM owner + MMA issuer: tcgen05.mma.kind::f16, A = h tile from TMEM (128 lanes x H/2 cols),
//                B = W stage (smem descriptor), D = fp32 accumulator 128 x 128 in TMEM (two buffers)
//   warps 4-11   epilogue, two groups of 4 (group g drains half the columns of every accumulator buffer): tcgen05.ld (thread = row), + bias,
//                online max / sum of exp over V, gathers z[blank] and z[y_u]; group 0 merges group 1's
//                partials and writes lse and (X_b, X_y) like K1
//   warps 12-19  A builders: tanh(f + g) of the NEXT tile into a shared-memory staging buffer while the
//                MMAs of the current tile run; once those complete, one tcgen05.st pass moves it into TMEM
// TMEM: A [0, 256) columns, kAccBufs = 2 accumulators of 128 columns in [256, 512).  (N = 64 with four
// buffers was measured slower: 2.20 vs 1.77 ms at c3 / H = 512 -- the narrower MMAs lose more than the
// deeper buffering gains.)  mbarriers link the roles.
// The training step's backward first pass on the forward's stored h is a separate kernel, k6_dz_2sm (below):
// A from shared memory by TMA, four accumulators, 16 dz epilogue warps.
// Constraints: H % 128 == 0, H <= 512 (any V: the last N tile's missing columns are masked).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>

#include "common.cuh"
#include "elem.cuh"
#include "joint.cuh"
#include "rnnt_b200.h"
#include "tc.cuh"

namespace rnnt {
namespace {

constexpr int kRowsPerTile = 128;
constexpr int kNTile = 128;      // accumulator columns per MMA (N)
constexpr int kAccBufs = 2;      // accumulator buffers in TMEM (kAccBufs * kNTile = 256 columns)
constexpr int kKBlock = 64;      // K per W stage (128 B of bf16: one SWIZZLE_128B row)
constexpr int kStageBytes = kNTile * kKBlock * 2;
constexpr int kThreads = 640;  // 20 warps: TMA, MMA, 2 spare, 2 x 4 epilogue, 8 builders
constexpr int kMaxStages = 16;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCol0 = 256;

// One K block (64 = 4 x K16) of D[tmem] (+)= A[tmem] . B[smem]^T, M = 128, N = kNTile, bf16 in, fp32
// accumulate: the four MMAs in one asm block so that the operands reach the uniform datapath once (per-MMA
// asm statements cost ~15 issue slots each in ELECT / R2UR conversions, as much as the MMA itself takes).
// A advances 8 TMEM columns (16 bf16) and the B descriptor 32 bytes (>> 4 = 2) per K16 step.  Called by the
// whole converged warp with warp-uniform operands; elect.sync picks the issuing lane.
__device__ __forceinline__ void mma_kblock(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, q, e;\n"
        ".reg .b32 a1, a2, a3;\n"
        ".reg .b64 b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 q, %4, %4;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u64 b1, %2, 2;\n"
        "add.u64 b2, %2, 4;\n"
        "add.u64 b3, %2, 6;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, q;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, q;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// The same K block as one pair MMA (cta_group::2, M = 256: the A rows are this CTA's tile then the peer's, each
// in its own TMEM at a_tmem; B's N = 128 columns are split 64 / 64 between the two CTAs' stages), issued by
// the pair's even CTA only.
__device__ __forceinline__ void mma_kblock_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, q, e;\n"
        ".reg .b32 a1, a2, a3;\n"
        ".reg .b64 b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 q, %4, %4;\n"
        "add.u32 a1, %1, 8;\n"
        "add.u32 a2, %1, 16;\n"
        "add.u32 a3, %1, 24;\n"
        "add.u64 b1, %2, 2;\n"
        "add.u64 b2, %2, 4;\n"
        "add.u64 b3, %2, 6;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, q;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], b2, %3, q;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a3], b3, %3, q;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// The pair K block with A from shared memory too (k6_dz_2sm): both descriptors advance 32 bytes (>> 4 = 2) per K16.
__device__ __forceinline__ void mma_kblock_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                  uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, q, e;\n"
        ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 q, %4, %4;\n"
        "add.u64 a1, %1, 2;\n"
        "add.u64 a2, %1, 4;\n"
        "add.u64 a3, %1, 6;\n"
        "add.u64 b1, %2, 2;\n"
        "add.u64 b2, %2, 4;\n"
        "add.u64 b3, %2, 6;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Instruction descriptor: fp32 D (bits 4-5 = 1), bf16 A (7-9 = 1) and B (10-12 = 1), both K-major,
// N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kNTile >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t kIdescPair = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kNTile >> 3) << 17) | (uint32_t(256 >> 4) << 24);
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// tanh on a pair, packed fp32x2 (FMUL2 / FADD2 / FFMA2) with MUFU ex2 and rcp:
//   tanh(x) = 1 - 2 / (1 + 2^(2 x log2 e)), signed: x -> +inf gives 1 - 2 rcp(inf) = 1, x -> -inf gives -1,
// so no |x|, no select and no copysign.  Absolute error ~2e-7 (the 1 - 2r cancellation near 0): relative error
// is large only where h is tiny, where a one-ulp bf16 difference in h moves z by ~1e-6 (R22).  The
// previous form (|x|, an odd series below 1/16, copysign) was ~1e-7 relative but cost 2.4x the FMA-pipe
// instructions: the builders are issue-bound, and K6 went 0.584 -> 0.518 ms at p124, 1.68 -> 1.60 ms at c3.
__device__ __forceinline__ float2 tanh2_mufu(float x0, float x1) {
    const float2 y = upk(fmul2(pk(x0, x1), pk(2.8853900817779268f, 2.8853900817779268f)));
    const float2 d = upk(fadd2(pk(ex2(y.x), ex2(y.y)), pk(1.f, 1.f)));
    return upk(ffma2(pk(rcp_approx(d.x), rcp_approx(d.y)), pk(-2.f, -2.f), pk(1.f, 1.f)));
}
// The same tanh with the reciprocal on the FMA pipe instead of MUFU: the builders' two MUFU ops per element
// and the epilogue's ex2 per logit share one MUFU pipe (16 results / clk / SM; ncu at p124: 64 % busy), which
// weighs on K6's pace at small V (one MUFU op less per element, tanh.approx, was 20 % faster at p124).  r0 = 0x7EF311C3 - bits(d) is within 5 %
// of 1 / d on d in [1, 2^64 + 1] (y clamped at 64 so d stays finite and r0 positive; the clamp is a compare and
// select, not fminf, so that a NaN input stays NaN as in the MUFU form), three Newton steps r += r (1 - d r)
// bring it to 9e-8 relative: |tanh error| 2.3e-7, as the MUFU form's.
__device__ __forceinline__ float2 tanh2_newton(float x0, float x1) {
    const float2 y = upk(fmul2(pk(x0, x1), pk(2.8853900817779268f, 2.8853900817779268f)));
    const float2 d = upk(fadd2(pk(ex2(y.x > 64.f ? 64.f : y.x), ex2(y.y > 64.f ? 64.f : y.y)), pk(1.f, 1.f)));
    const float2 nd = make_float2(-d.x, -d.y);
    float2 r = make_float2(__int_as_float(0x7EF311C3 - __float_as_int(d.x)),
                           __int_as_float(0x7EF311C3 - __float_as_int(d.y)));
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float2 e = upk(ffma2(pk(nd.x, nd.y), pk(r.x, r.y), pk(1.f, 1.f)));
        r = upk(ffma2(pk(r.x, r.y), pk(e.x, e.y), pk(r.x, r.y)));
    }
    return upk(ffma2(pk(r.x, r.y), pk(-2.f, -2.f), pk(1.f, 1.f)));
}
// words (of the 4 per 16-byte item) whose tanh takes the Newton reciprocal in the loss-only forward; the rest
// use MUFU rcp.  A/B (scripts/gpu_k6nr.sh, profiles/r02_g/k6nr.txt), K6 at p124: 0 words 0.414 ms, 1 word
// 0.4015, 2 words 0.411, 4 words 0.437 -- past one word the FMA-pipe work costs more than the MUFU time it
// frees.  The training step's forward (h stored from the builders) was 1 % slower with 1 word: it keeps MUFU.
#ifndef RNNT_K6_NR
#define RNNT_K6_NR 1
#endif
static_assert(RNNT_K6_NR >= 0 && RNNT_K6_NR <= 4, "Newton words per item");
// z[k] for a per-lane k in [0, 32) without local memory: a 5-level select tree (31 FSEL) instead of 32
// compare-and-move pairs.
__device__ __forceinline__ float select32(const float (&z)[32], int k) {
    float s[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = (k & 1) ? z[2 * i + 1] : z[2 * i];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = (k & 2) ? s[2 * i + 1] : s[2 * i];
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = (k & 4) ? s[2 * i + 1] : s[2 * i];
#pragma unroll
    for (int i = 0; i < 2; ++i) s[i] = (k & 8) ? s[2 * i + 1] : s[2 * i];
    return (k & 16) ? s[1] : s[0];
}
struct JointArgs {
    const __nv_bfloat16* f;
    const __nv_bfloat16* g;
    const float* bias;
    const int32_t* targets;
    const int32_t* T_b;
    const int32_t* U_b;
    int B, Tmax, Umax, H, V, blank;
    int64_t rows;  // B * Tmax * (Umax + 1)
    int stages;
    const int* rowmap;  // [rows] compact row -> padded row index b*Tmax*(Umax+1) + t*(Umax+1) + u (k6_rowmap)
    const int* nrows;   // number of valid cells (compact rows)
    int dbg;  // diagnostics (env RNNT_K6_DEBUG, never set in production): 1 = builders skip tanh (a timing
              // ablation on the builders' slow path: wrong losses), 4 = per-role barrier-wait cycle counters
              // printed to stderr.  (No switch inside the hot loops: runtime selects in the builders' loop cost
              // ~10 % at p124; the tanh.approx opt-in, the load / epilogue-math ablations and k6_dz_2sm's
              // per-lane dz-store A/B measured that way are recorded in DESIGN.md and removed.)
    unsigned long long* prof;
    float* lse_out;
    double2* lp_out;
    // backward pass (kGrad): the forward's lse / lp and K2's alpha / beta / logP in, dz and h out
    const float* lse_in;
    const double2* lp_in;
    const double* alpha;
    const double* beta;
    const double* logp;
    const float* grad_scale;
    __nv_bfloat16* dz_out;  // [rows][Vp] row-major, Vp = V rounded up to whole N tiles (tail columns 0)
    __nv_bfloat16* h_out;   // [rows][H]: h stored by the builders (the training step's forward; K6<grad> A/B), or null
    const __nv_bfloat16* h_in;  // K6<grad> only: [rows][H] h as the forward stored it -- loaded, not recomputed
                                // (k6_dz_2sm reads it through its own tensor map; k6_joint_lse<true> by bulk copies)
};

// Per-row scalars of dz for cell (t,u) of utterance b: the occupancies of the two scored arcs leaving it, as K3
// (k3_grad.cu), times grad_scale[b]; padded rows and invalid / no-path utterances (logP not finite) get gl = false
// (dz = 0).  lsel = lse log2 e (+inf for an all -inf row: p = 0).
struct DzRow {
    bool gl;
    float sb, sy, lsel;
    int gy;  // the label column, -1 if none
};
__device__ __forceinline__ DzRow dz_row(const JointArgs& a, bool in, int b, int t, int u, int T, int U, bool live,
                                        int yv, int64_t cells) {
    DzRow d{false, 0.f, 0.f, INFINITY, -1};
    const double lP = in ? a.logp[b] : 0.0;
    d.gl = live && isfinite(lP);
    if (!d.gl) return d;
    const int Up1 = a.Umax + 1;
    const int64_t dcell = (static_cast<int64_t>(b) * (a.Tmax + a.Umax) + (t + u)) * Up1 + u;
    const float lse = a.lse_in[static_cast<int64_t>(b) * cells + t * Up1 + u];
    const double2 l = a.lp_in[dcell];
    const double al = a.alpha[dcell];
    if (t < T - 1)
        d.sb = __expf(static_cast<float>(al + l.x + a.beta[dcell + Up1] - lP));
    else if (u == U)
        d.sb = __expf(static_cast<float>(al + l.x - lP));
    if (u < U) {
        d.sy = __expf(static_cast<float>(al + l.y + a.beta[dcell + Up1 + 1] - lP));
        d.gy = yv;
    }
    if (a.grad_scale) {
        const float sc = a.grad_scale[b];
        d.sb *= sc;
        d.sy *= sc;
    }
    d.lsel = (lse == -INFINITY) ? INFINITY : lse * kLog2e;
    return d;
}

// One 32-column chunk v0 .. v0 + 31 of this thread's dz row (K3's formula on z = acc + bias, k3_grad.cu):
// dz = bf16(2^(z log2 e - lse log2 e) gam - [v = blank] sb - [v = y] sy), zeros where the row carries no
// gradient (!gl).  Through the warp's 2 KB staging block at `st`: each lane writes its row's 4 chunks, then reads
// back (row = lane / 4 + 8 s, chunk = lane % 4) so that every global store instruction writes 8 whole 64-byte row
// segments (8 L1 wavefronts instead of 32 for thread-per-row stores).  row0: the compact row of lane 0; rows:
// the valid rows; ldz: dz's row pitch in elements.  dz_map (k6_dz_2sm): the staging block's layout is TMA's
// SWIZZLE_64B one, so lane 0 stores it with one TMA tile store (box {32 columns, 32 rows}) instead of the warp's
// 4 x 16-byte loads and stores per lane -- half the L1 traffic; the block is reused once that store has read it.
template <bool kSB>
__device__ __forceinline__ void dz_chunk(const JointArgs& a, const uint32_t (&r)[32], const float* sbias,
                                         const float4 (&bq)[8], int v0, bool gl, f32x2 l2, f32x2 nl, f32x2 g2,
                                         float sb, float sy, int gy, uint32_t st, int lane, int64_t row0,
                                         int64_t rows, int64_t ldz, const CUtensorMap* dz_map = nullptr) {
    float g[32];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float4 bb = kSB ? reinterpret_cast<const float4*>(sbias + v0)[j] : bq[j];
        const f32x2 z0 = fadd2(pk(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])), pk(bb.x, bb.y));
        const f32x2 z1 = fadd2(pk(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])), pk(bb.z, bb.w));
        const float2 p0 = upk(fmul2(ex2x2(ffma2(z0, l2, nl)), g2));
        const float2 p1 = upk(fmul2(ex2x2(ffma2(z1, l2, nl)), g2));
        g[4 * j] = p0.x;
        g[4 * j + 1] = p0.y;
        g[4 * j + 2] = p1.x;
        g[4 * j + 3] = p1.y;
    }
    if (static_cast<unsigned>(a.blank - v0) < 32u) {  // the arcs' own logits
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (v0 + j == a.blank) g[j] -= sb;
    }
    if (static_cast<unsigned>(gy - v0) < 32u) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (v0 + j == gy) g[j] -= sy;
    }
    if (dz_map && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();  // the previous chunk's reads (or TMA store) are done
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        const uint32_t w0 = gl ? pack_bf16x2(g[8 * q4 + 0], g[8 * q4 + 1]) : 0u;
        const uint32_t w1 = gl ? pack_bf16x2(g[8 * q4 + 2], g[8 * q4 + 3]) : 0u;
        const uint32_t w2 = gl ? pack_bf16x2(g[8 * q4 + 4], g[8 * q4 + 5]) : 0u;
        const uint32_t w3 = gl ? pack_bf16x2(g[8 * q4 + 6], g[8 * q4 + 7]) : 0u;
        const uint32_t ad = st + lane * 64u + ((q4 ^ ((lane >> 1) & 3)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                     : "memory");
    }
    if (dz_map) {  // rows past `rows` (< R: dz's allocation) get zeros; TMA clips at R
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && row0 < rows) tma_store_2d(dz_map, st, v0, static_cast<int>(row0));
        return;
    }
    __syncwarp();
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
        const int rr = (lane >> 2) + 8 * s4, kk = lane & 3;
        uint4 o;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w)
                     : "r"(st + rr * 64u + ((kk ^ ((rr >> 1) & 3)) << 4))
                     : "memory");
        const int64_t orow = row0 + rr;
        if (orow < rows) *reinterpret_cast<uint4*>(a.dz_out + orow * ldz + v0 + kk * 8) = o;
    }
}

// kGrad = false: the forward (lse + gathers).  kGrad = true: the backward's first pass -- the same GEMM
// recomputes z and the epilogue forms dz = softmax(z) (occ_b + occ_y) - [v = blank] occ_b - [v = y] occ_y
// (K3's formula, with the forward's lse and K2's alpha / beta), stored in bf16 for the two backward GEMMs.
// h = bf16(tanh(f + g)): the builders store it when h_out is set (the training step's forward; or K6<grad>
// itself), and K6<grad> with h_in loads the forward's rows instead of recomputing them (K6<grad> 601 -> 457 us
// at p124, 1791 -> 1651 us at c3; the forward +20 us for the stores: the builders' MUFU work was K6<grad>'s
// limit at p124).
// kCl = 2: CTA pairs (clusters of 2) share every W stage -- each CTA fetches half of the stage's rows and
// multicasts it into both CTAs' shared memory (half the W traffic from L2 per SM); the pair walks the same
// W sequence in lockstep (a stage is refilled once both MMAs released it) and the same number of row tiles
// (the second CTA's last one may be a dummy past the end).
constexpr int kSBiasMaxV = 4096;  // largest V whose bias is staged in shared memory (16 KB)

// bias(v..v+3) from global memory (read-only path; 16-byte aligned, checked by joint_front).  Columns past V
// (the last N tile's tail, where TMA zero-fills W's missing rows) get -inf: absent from the max and the sum,
// so V need not be a multiple of the tile.  Warp-uniform branch (v depends only on the column chunk).
__device__ __forceinline__ float4 bias4(const JointArgs& a, int v) {
    if (v + 4 <= a.V) return a.bias ? __ldg(reinterpret_cast<const float4*>(a.bias + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
    float f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = v + k < a.V ? (a.bias ? __ldg(a.bias + v + k) : 0.f) : -INFINITY;
    return make_float4(f[0], f[1], f[2], f[3]);
}

// kSB: the bias (padded to whole N tiles with -inf) is staged once in shared memory -- when it is small
// (Vp <= kSBiasMaxV); else it is read per chunk from global memory (bias4), issued ahead of the TMEM load.
// Measured: the shared copy is ~14% faster on the forward at V = 1024 (epilogue latency).
// kPair (kCl = 2): the pair's tiles go through ONE pair MMA (cta_group::2, M = 256) per K16 step instead of one
// MMA per CTA, each CTA holding only its 64-column half of every W stage (no multicast): per CTA and stage 8 KB
// of W against 256 MMA cycles, half of what the multicast pair receives -- the L2 -> SM delivery (~47 B per
// cycle per SM measured on K9) is then no longer the limit.  Only the even CTA issues MMAs; the odd CTA's
// builders tell it that their A tile is in TMEM (one remote arrive per tile) and its epilogue warps release the
// accumulators on the leader's acc_empty (one remote arrive per warp per N tile).
// kStore (forward only): the builders also store h for the training step's K6<grad> (a compile-time choice: the
// store and its predicate stay out of the loss-only forward's builder loop).
template <bool kGrad, int kCl, bool kSB, bool kPair, bool kStore = false>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kThreads, 1)
    k6_joint_lse(const __grid_constant__ CUtensorMap w_map, const JointArgs a) {
    static_assert(!kPair || kCl == 2, "pair MMAs need clusters of 2");
    constexpr int kSlot = kPair ? kStageBytes / 2 : kStageBytes;  // a W stage slot in this CTA
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // carve: [W stages (1024-aligned)] [A staging 128 x H bf16] [epilogue exchange] [barriers] [tmem slot]
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* wst = base;
    uint8_t* stage_a = wst + static_cast<size_t>(a.stages) * kSlot;
    const int Vp = (a.V + kNTile - 1) / kNTile * kNTile;  // V rounded up to whole N tiles
    // A staging: 128 rows of H + kJointHPad bf16 (the 16-byte pad: conflict-free thread-per-row reads; h_in: the
    // forward's h rows land in the first H columns by one bulk copy each)
    float* sbias = reinterpret_cast<float*>(stage_a + static_cast<size_t>(kRowsPerTile) * (a.H + kJointHPad) * 2);
    float4* xchg = reinterpret_cast<float4*>(sbias + (kSB ? Vp : 0));  // [2][128] epilogue group 1 -> 0 partials
    uint64_t* bars = reinterpret_cast<uint64_t*>(xchg + 2 * kRowsPerTile);
    uint64_t* b_full = bars;                   // [stages]
    uint64_t* b_empty = bars + kMaxStages;     // [stages]
    uint64_t* a_full = bars + 2 * kMaxStages;
    uint64_t* a_empty = a_full + 1;
    uint64_t* acc_full = a_full + 2;                 // [kAccBufs]
    uint64_t* acc_empty = a_full + 2 + kAccBufs;     // [kAccBufs]
    uint64_t* h_full = a_full + 2 + 2 * kAccBufs;    // h_in: the tile's h rows have landed in the staging buffer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_full + 1);
    // kGrad: per epilogue warp, a 32-row x 32-column bf16 dz staging block (2 KB), 16-byte chunks XOR-swizzled
    uint8_t* dzst = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 127) & ~uintptr_t(127));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int H = a.H, V = a.V;
    if (kSB)  // read by the epilogue only, after the __syncthreads of the setup below
        for (int i = threadIdx.x; i < Vp; i += blockDim.x) sbias[i] = i < V ? (a.bias ? a.bias[i] : 0.f) : -INFINITY;
    const int KB = H / kKBlock, NT = Vp / kNTile;
    const int64_t rows = *a.nrows;  // valid cells only: padding costs no GEMM work
    const int64_t ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
    const int64_t cells = static_cast<int64_t>(a.Tmax) * (a.Umax + 1);
    // compact row -> (b, t, u); false past the last row
    auto decode = [&](int64_t row, int& b, int& t, int& u) -> bool {
        if (row >= rows) return false;
        const int p = __ldg(a.rowmap + row);
        b = static_cast<int>(p / cells);
        const int rem = static_cast<int>(p - static_cast<int64_t>(b) * cells);
        t = rem / (a.Umax + 1);
        u = rem - t * (a.Umax + 1);
        return true;
    };

    const uint32_t crank = kCl > 1 ? cluster_rank() : 0;
    const bool leader = crank == 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], kPair ? 1 : kCl);  // released by the MMAs of every CTA of the cluster
        }
        mbar_init(a_full, kPair ? 256 + 1 : 256);  // pair: + the odd CTA's builders (one remote arrive)
        mbar_init(a_empty, 1);
        mbar_init(h_full, 1);
        for (int i = 0; i < kAccBufs; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], kPair ? 256 + 8 : 256);  // both epilogue groups (pair: + the odd CTA's 8 warps)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&w_map)) : "memory");
    }
    if (warp == 1) {
        if constexpr (kPair) {
            tmem_alloc_2sm(tmem_slot, kTmemCols);
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(kTmemCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();  // barriers initialised cluster-wide before any multicast signals them
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // Row tiles: blockIdx.x + k * gridDim.x for k < n_iter, n_iter taken from the cluster's first CTA
    const int64_t bx = blockIdx.x, cl0 = bx - bx % kCl;
    const int64_t n_iter = ntiles > cl0 ? (ntiles - cl0 + gridDim.x - 1) / gridDim.x : 0;
    const bool pon = (a.dbg & 4) != 0;
    unsigned long long w_tma = 0, w_afull = 0, w_accempty = 0, w_bfull = 0, w_accfull = 0, w_aempty = 0;
    const long long t_start = clock64();

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < n_iter; ++k)
                for (int n = 0; n < NT; ++n)
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait_t(&b_empty[s], ph ^ 1, pon, w_tma);
                        if constexpr (kPair) {  // own 64-column half, landing on the leader's barrier
                            if (leader) mbar_expect_tx(&b_full[s], kStageBytes);  // both halves
                            tma_load_2d_2sm(wst + static_cast<size_t>(s) * kSlot, &w_map, leader_addr(&b_full[s]),
                                            kb * kKBlock, n * kNTile + static_cast<int>(crank) * (kNTile / 2));
                        } else {
                        mbar_expect_tx(&b_full[s], kStageBytes);  // the whole stage lands here (both halves)
                        if constexpr (kCl > 1)
                            tma_load_2d_mc(wst + static_cast<size_t>(s) * kStageBytes + crank * (kStageBytes / kCl),
                                           &w_map, &b_full[s], kb * kKBlock, n * kNTile + crank * (kNTile / kCl),
                                           static_cast<uint16_t>((1u << kCl) - 1));
                        else
                            tma_load_2d(wst + static_cast<size_t>(s) * kStageBytes, &w_map, &b_full[s], kb * kKBlock,
                                        n * kNTile);
                        }
                        if (++s == a.stages) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
        }
    } else if (warp == 1 && (!kPair || leader)) {
        // ===== MMA issuer (pair: the even CTA, for both) =====
        int s = 0;
        uint32_t ph = 0;
        uint32_t it = 0;  // accumulator use counter
        uint32_t tl = 0;  // local tile counter
        for (int64_t k = 0; k < n_iter; ++k, ++tl) {
            mbar_wait_t(a_full, tl & 1, pon, w_afull);
            tc_fence_after();
            for (int n = 0; n < NT; ++n, ++it) {
                const uint32_t acc = it % kAccBufs;
                mbar_wait_t(&acc_empty[acc], ((it / kAccBufs) & 1) ^ 1, pon, w_accempty);
                tc_fence_after();
                const uint32_t d_tmem = tmem + kAccCol0 + acc * kNTile;
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait_t(&b_full[s], ph, pon, w_bfull);
                    tc_fence_after();
                    const uint64_t bdesc = sw128_desc(smem_u32(wst + static_cast<size_t>(s) * kSlot));
                    if constexpr (kPair)
                        mma_kblock_2sm(d_tmem, tmem + kb * (kKBlock / 2), bdesc, kIdescPair, kb ? 1u : 0u);
                    else
                        mma_kblock(d_tmem, tmem + kb * (kKBlock / 2), bdesc, kIdesc, kb ? 1u : 0u);
                    // frees the W stage (in every CTA of the cluster: its producer refills both) once these MMAs complete
                    if constexpr (kPair)
                        tc_commit_2sm_mc(&b_empty[s], 3);
                    else if constexpr (kCl > 1)
                        tc_commit_mc(&b_empty[s], static_cast<uint16_t>((1u << kCl) - 1));
                    else
                        tc_commit(&b_empty[s]);
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if constexpr (kPair)
                    tc_commit_2sm_mc(&acc_full[acc], 3);
                else
                    tc_commit(&acc_full[acc]);
            }
            // the A tile in TMEM may be overwritten.  (Handing it over per K half, so that the copy of half 0
            // overlaps the last N tile's MMAs on half 1, measured slower: 1.60 vs 1.52 ms.)
            if constexpr (kPair)
                tc_commit_2sm_mc(a_empty, 3);
            else
                tc_commit(a_empty);
        }
    } else if (warp >= 4 && warp < 12) {
        // ===== epilogue: thread = row; both groups drain every accumulator buffer, group eg taking columns
        // [eg * N/2, (eg + 1) * N/2) of each N tile, so a buffer is free after half an N tile's work (with
        // whole N tiles alternating between the groups, the drain took ~1.4x the MMA time and the MMA waited
        // on it: 1.65 vs 1.52 ms); per tile, group 1 hands its row partials (max, sum, z[blank], z[y]) to
        // group 0 through shared memory, which finishes the row =====
        const int q = warp & 3, eg = (warp - 4) >> 2;
        const int rl = q * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t it = 0, tile_local = 0;
        for (int64_t k = 0; k < n_iter; ++k) {
            const int64_t tile = bx + k * gridDim.x;
            int b = 0, t = 0, u = 0;
            const bool in = decode(tile * kRowsPerTile + rl, b, t, u);
            const int T = in ? min(a.T_b[b], a.Tmax) : 0, U = in ? min(a.U_b[b], a.Umax) : 0;
            const bool live = in && t < T && u <= U;
            const int yv = (live && u < U) ? a.targets[static_cast<int64_t>(b) * a.Umax + u] : -1;
            if constexpr (kGrad) {
                const DzRow d = dz_row(a, in, b, t, u, T, U, live, yv, cells);
                const bool gl = d.gl;
                const float sb = d.sb, sy = d.sy, gam = d.sb + d.sy, lsel = d.lsel;
                const int gy = d.gy;
                const f32x2 l2 = pk(kLog2e, kLog2e), nl = pk(-lsel, -lsel), g2 = pk(gam, gam);
                for (int n = 0; n < NT; ++n, ++it) {
                    const uint32_t acc = it % kAccBufs;
                    mbar_wait_t(&acc_full[acc], (it / kAccBufs) & 1, pon, w_accfull);
                    tc_fence_after();
#pragma unroll 1
                    for (int c = eg * (kNTile / 64); c < (eg + 1) * (kNTile / 64); ++c) {
                        const int v0 = n * kNTile + c * 32;
                        float4 bq[8];  // !kSB: global bias loads in flight under the TMEM load
#pragma unroll
                        for (int j = 0; j < 8; ++j) bq[j] = kSB ? make_float4(0.f, 0.f, 0.f, 0.f) : bias4(a, v0 + 4 * j);
                        uint32_t r[32];
                        TMEM_LD32(lane_base + kAccCol0 + acc * kNTile + c * 32, r);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (c + 1 == (eg + 1) * (kNTile / 64)) {
                            // this group's last load of the buffer: release it now, before this chunk's dz math and
                            // stores (the MMA was waiting ~25 % of its time on the buffer otherwise)
                            tc_fence_before();
                            if (!kPair || leader) {
                                mbar_arrive(&acc_empty[acc]);
                            } else {  // the odd CTA: one arrive per warp on the leader's barrier
                                __syncwarp();
                                if (lane == 0) mbar_arrive_remote(&acc_empty[acc], 0);
                            }
                        }
                        dz_chunk<kSB>(a, r, sbias, bq, v0, gl, l2, nl, g2, sb, sy, gy,
                                      smem_u32(dzst) + static_cast<uint32_t>(warp - 4) * 2048u, lane,
                                      tile * kRowsPerTile + q * 32, rows, static_cast<int64_t>(NT) * kNTile);
                    }
                }
                continue;
            }
            float m = -INFINITY, ssum = 0.f, zb = 0.f, zy = 0.f;
            for (int n = 0; n < NT; ++n, ++it) {
                const uint32_t acc = it % kAccBufs;
                mbar_wait_t(&acc_full[acc], (it / kAccBufs) & 1, pon, w_accfull);
                tc_fence_after();
#pragma unroll 1
                for (int c = eg * (kNTile / 64); c < (eg + 1) * (kNTile / 64); ++c) {  // group eg: half the columns
                    const int v0 = n * kNTile + c * 32;
                    float4 bq[8];  // !kSB: global bias loads in flight under the TMEM load
#pragma unroll
                    for (int j = 0; j < 8; ++j) bq[j] = kSB ? make_float4(0.f, 0.f, 0.f, 0.f) : bias4(a, v0 + 4 * j);
                    uint32_t r[32];
                    TMEM_LD32(lane_base + kAccCol0 + acc * kNTile + c * 32, r);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (c + 1 == (eg + 1) * (kNTile / 64)) {  // the group's last load: release the buffer now
                        tc_fence_before();
                        if (!kPair || leader) {
                            mbar_arrive(&acc_empty[acc]);
                        } else {  // the odd CTA: one arrive per warp on the leader's barrier
                            __syncwarp();
                            if (lane == 0) mbar_arrive_remote(&acc_empty[acc], 0);
                        }
                    }
                    f32x2 zz[16];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 bb = kSB ? reinterpret_cast<const float4*>(sbias + v0)[j] : bq[j];
                        zz[2 * j] = fadd2(pk(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1])), pk(bb.x, bb.y));
                        zz[2 * j + 1] =
                            fadd2(pk(__uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])), pk(bb.z, bb.w));
                    }
                    float cm = -INFINITY;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float2 v = upk(zz[j]);
                        cm = max3(cm, v.x, v.y);
                    }
                    const float mn = fmaxf(m, cm);
                    if (mn == -INFINITY) continue;  // nothing finite yet (a chunk of masked tail columns)
                    const f32x2 l2 = pk(kLog2e, kLog2e), nml = pk(-mn * kLog2e, -mn * kLog2e);
                    f32x2 accs[4] = {pk(0.f, 0.f), pk(0.f, 0.f), pk(0.f, 0.f), pk(0.f, 0.f)};
#pragma unroll
                    for (int j = 0; j < 16; ++j) accs[j & 3] = fadd2(accs[j & 3], ex2x2(ffma2(zz[j], l2, nml)));
                    const float2 a2s = upk(fadd2(fadd2(accs[0], accs[1]), fadd2(accs[2], accs[3])));
                    ssum = fmaf(ssum, ex2((m - mn) * kLog2e), a2s.x + a2s.y);
                    m = mn;
                    float z[32];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float2 v = upk(zz[j]);
                        z[2 * j] = v.x;
                        z[2 * j + 1] = v.y;
                    }
                    if (static_cast<unsigned>(a.blank - v0) < 32u) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (v0 + j == a.blank) zb = z[j];
                    }
                    if (static_cast<unsigned>(yv - v0) < 32u) zy = select32(z, yv - v0);  // some lane's label is in most chunks
                }
            }
            float4* xb_ = xchg + (tile_local & 1) * kRowsPerTile + rl;
            if (eg == 1) *xb_ = make_float4(m, ssum, zb, zy);
            asm volatile("bar.sync 3, 256;" ::: "memory");  // the two epilogue groups
            ++tile_local;
            if (eg == 1) continue;
            {
                const float4 o = *xb_;
                const float mm = fmaxf(m, o.x);
                ssum = (mm == -INFINITY) ? 0.f : ssum * ex2((m - mm) * kLog2e) + o.y * ex2((o.x - mm) * kLog2e);
                m = mm;
                zb += o.z;  // the column's owner set it; the other group left 0
                zy += o.w;
            }
            if (live) {
                const float lse = m + lg2(ssum) * kLn2;
                const int64_t urow = static_cast<int64_t>(b) * cells + t * (a.Umax + 1) + u;
                a.lse_out[urow] = lse;
                const bool ybad = (u < U) && (yv < 0 || yv >= a.V || yv == a.blank);
                float xb = zb - lse;
                float xy = (u < U) ? (ybad ? __int_as_float(0x7fc00000) : zy - lse) : -INFINITY;
                if (lse != lse) {  // a NaN in the row: +inf arc scores (common.cuh kNanArc)
                    xb = INFINITY;
                    xy = (u < U) ? INFINITY : -INFINITY;
                }
                const int64_t diag = static_cast<int64_t>(b) * (a.Tmax + a.Umax) + (t + u);
                a.lp_out[diag * (a.Umax + 1) + u] = make_double2(xb, xy);
            }
        }
    } else if (warp >= 12) {
        // ===== A builders: warp -> (row quarter q, K half kh) =====
        // Build: lane = 16-byte K chunk, so each load instruction reads contiguous bytes of one row (coalesced;
        // consecutive rows mostly share the f row).  Copy to TMEM: thread = row (tcgen05.st lane quarter).
        const int q = warp & 3, kh = (warp - 12) >> 2;
        const int rl = q * 32 + lane;
        const int nch = H / 16;            // 16-byte chunks per K half
        const int row_bytes = (H + kJointHPad) * 2;  // +16 B: conflict-free row reads without a swizzle
        uint8_t* my_row = stage_a + static_cast<size_t>(rl) * row_bytes;
        const uint32_t sa_base = smem_u32(stage_a);  // 32-bit shared addresses for the builders' stores
                const uint4* f4 = reinterpret_cast<const uint4*>(a.f);
        const uint4* g4 = reinterpret_cast<const uint4*>(a.g);
        const int items = 32 * nch;        // (row of the quarter, chunk of the half)
        // Row-map entry of this lane's row (q*32 + lane) in a tile, -1 past the end; fetched one build ahead so
        // its latency does not start each build.
        const bool identity = rows == a.rows;  // no padding: the map is the identity, skip its loads
        auto map_of = [&](int64_t tile) -> int {
            const int64_t row = tile * kRowsPerTile + rl;
            if (tile >= ntiles || row >= rows) return -1;
            return identity ? static_cast<int>(row) : __ldg(a.rowmap + row);
        };
        int p_next = -1;
        const bool hstore = kGrad ? a.h_out != nullptr : kStore, hload = kGrad && a.h_in != nullptr;
        auto build = [&](int64_t tile, int p) {
            if (hload) {
                // h as the training step's forward stored it: one bulk async copy per row into the staging
                // buffer (warps 12-15, one row per thread), completing on h_full; no tanh here.  All 8 builder
                // warps have copied the previous tile from the staging buffer into TMEM (bar.sync) first.
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 4, 256;" ::: "memory");
                if (warp < 16) {
                    const int64_t nv = std::max<int64_t>(0, std::min<int64_t>(kRowsPerTile, rows - tile * kRowsPerTile));
                    if (warp == 12 && lane == 0) mbar_expect_tx(h_full, static_cast<uint32_t>(nv * H * 2));
                    const int r = (warp - 12) * 32 + lane;
                    if (r < nv)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                sa_base + static_cast<uint32_t>(r * row_bytes)),
                            "l"(a.h_in + (tile * kRowsPerTile + r) * H), "r"(static_cast<uint32_t>(H * 2)),
                            "r"(smem_u32(h_full))
                            : "memory");
                }
                return;
            }
            // lane r: chunk offsets (16-byte units) of row q*32 + r's f and g rows, -1 past the end
            int fo = -1, go = -1;
            if (p >= 0) {
                const int b = static_cast<int>(p / cells);
                const int rem = static_cast<int>(p - static_cast<int64_t>(b) * cells);
                const int t = rem / (a.Umax + 1), u = rem - t * (a.Umax + 1);
                fo = (b * a.Tmax + t) * (H / 8) + kh * nch;
                go = (b * (a.Umax + 1) + u) * (H / 8) + kh * nch;
            }
            // items = 32 nch is a multiple of 4 * 32 (nch in {8, 16, 24, 32}): every batch is full
            // fast: the tile has no rows past the end and no diagnostics -> no per-item / per-word selects
            const bool fast = (tile + 1) * kRowsPerTile <= rows && (a.dbg & 1) == 0;  // no-tanh ablation: slow path
            auto batch = [&](const int (&rows_)[4], const int (&cs)[4], auto fast_c) {
                constexpr bool kFast = decltype(fast_c)::value;
                uint4 fa[4], ga[4];
                bool ok[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int fro = __shfl_sync(0xffffffffu, fo, rows_[j] & 31);
                    const int gro = __shfl_sync(0xffffffffu, go, rows_[j] & 31);
                    ok[j] = kFast || fro >= 0;
                    // unconditional loads (row 0 stands in past the end; its output is zeroed below): no
                    // per-register zero fill; 32-bit indices: one IMAD.WIDE per load
                    fa[j] = __ldg(f4 + static_cast<uint32_t>((kFast || ok[j] ? fro : 0) + cs[j]));
                    ga[j] = __ldg(g4 + static_cast<uint32_t>((kFast || ok[j] ? gro : 0) + cs[j]));
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t fw[4] = {fa[j].x, fa[j].y, fa[j].z, fa[j].w};
                    const uint32_t gw[4] = {ga[j].x, ga[j].y, ga[j].z, ga[j].w};
                    uint32_t ow[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 x = unpack_bf16x2(fw[e]), y = unpack_bf16x2(gw[e]);
                        const float2 xs = upk(fadd2(pk(x.x, x.y), pk(y.x, y.y)));
                        constexpr int kNR = (kGrad || kStore) ? 0 : RNNT_K6_NR;
                        const float2 h = e < 4 - kNR ? tanh2_mufu(xs.x, xs.y) : tanh2_newton(xs.x, xs.y);
                        ow[e] = kFast ? pack_bf16x2(h.x, h.y)
                                      : !ok[j] ? 0u : (a.dbg & 1) ? (fw[e] ^ gw[e]) : pack_bf16x2(h.x, h.y);
                    }
                    const int r2 = q * 32 + rows_[j];
                    const int cg = kh * nch + cs[j];
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sa_base + r2 * row_bytes + (cg << 4)),
                                 "r"(ow[0]), "r"(ow[1]), "r"(ow[2]), "r"(ow[3])
                                 : "memory");
                    // h for K6<grad> / K8 / K9 / K7, straight from registers: a warp's store writes 512 contiguous
                    // bytes of one row at H = 512 (a bulk copy per row from the staging buffer made the next build
                    // wait for the copy to read it: p124 forward 495 -> 582 us)
                    if (hstore && (kFast || ok[j]))
                        *reinterpret_cast<uint4*>(a.h_out + (tile * kRowsPerTile + r2) * H + cg * 8) =
                            make_uint4(ow[0], ow[1], ow[2], ow[3]);
                }
            };
            if (nch == 32) {  // H = 512: lane = chunk, item j of a batch = row i0 / 32 + j
                for (int i0 = 0; i0 < items; i0 += 4 * 32) {
                    const int r0 = i0 >> 5;
                    const int rows_[4] = {r0, r0 + 1, r0 + 2, r0 + 3}, cs[4] = {lane, lane, lane, lane};
                    if (fast)
                        batch(rows_, cs, std::true_type{});
                    else
                        batch(rows_, cs, std::false_type{});
                }
            } else {
                int rr = lane / nch, c = lane - (lane / nch) * nch;  // this lane's first item
                const int drr = 32 / nch, dc = 32 - drr * nch;        // item += 32
                for (int i0 = 0; i0 < items; i0 += 4 * 32) {
                    int rows_[4], cs[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        rows_[j] = rr;
                        cs[j] = c;
                        rr += drr;
                        c += dc;
                        if (c >= nch) {
                            c -= nch;
                            ++rr;
                        }
                    }
                    if (fast)
                        batch(rows_, cs, std::true_type{});
                    else
                        batch(rows_, cs, std::false_type{});
                }
            }
            __syncwarp();  // each thread copies its own row, written by the whole warp
        };
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t tl = 0;
        if (n_iter > 0) {
            const int p0 = map_of(bx);
            p_next = map_of(bx + gridDim.x);
            build(bx, p0);
        }
        for (int64_t k = 0; k < n_iter; ++k, ++tl) {
            const int64_t tile = bx + k * gridDim.x;
            if (tl > 0) mbar_wait_t(a_empty, (tl - 1) & 1, pon, w_aempty);
            if (hload) mbar_wait(h_full, tl & 1);
            tc_fence_after();
            // staging -> TMEM: this thread's row, its K half = nch chunks = nch * 4 columns
            for (int c0 = 0; c0 < nch; c0 += 8) {
                uint32_t r[32];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int cg = kh * nch + c0 + i;
                    const uint4 v = *reinterpret_cast<const uint4*>(my_row + (cg << 4));
                    r[4 * i + 0] = v.x;
                    r[4 * i + 1] = v.y;
                    r[4 * i + 2] = v.z;
                    r[4 * i + 3] = v.w;
                }
                TMEM_ST32(lane_base + static_cast<uint32_t>((kh * nch + c0) * 4), r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            if (!kPair || leader) {
                mbar_arrive(a_full);
            } else {  // the odd CTA's builders: all 256 done, then one arrive on the leader's barrier
                asm volatile("bar.sync 5, 256;" ::: "memory");
                if (warp == 12 && lane == 0) mbar_arrive_remote(a_full, 0);
            }
            if (k + 1 < n_iter) {
                const int p = p_next;
                p_next = map_of(tile + 2 * static_cast<int64_t>(gridDim.x));
                build(tile + gridDim.x, p);
            }
        }
    }
    if (pon && lane == 0) {
        unsigned long long* o = a.prof + static_cast<size_t>(blockIdx.x) * 8;
        const unsigned long long tot = clock64() - t_start;
        if (warp == 0) { o[0] = tot; o[1] = w_tma; }
        if (warp == 1) { o[2] = w_afull; o[3] = w_accempty; o[4] = w_bfull; }
        if (warp == 4) o[5] = w_accfull;
        if (warp == 8) o[7] = w_accfull;
        if (warp == 12) o[6] = w_aempty;
    }
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();  // no CTA leaves while its partner may still multicast into it
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        if constexpr (kPair)
            tmem_dealloc_2sm(tmem, kTmemCols);
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// K6<grad> with h given (the training step, whose forward stored h): the backward's first pass as a plain pair
// GEMM with both operands in shared memory.  A = the tile's 128 h rows as KB = H / 64 blocks of [128 x 64] bf16
// (SW128, one 2-SM TMA each onto the leader's barrier, freed block by block by the tile's last N tile so the next
// tile's rows stream in under it), B = the W stages as k6_joint_lse's pair path.  No warp builds A and A takes no
// TMEM, so the 512 TMEM columns hold four 128-column accumulators and 16 epilogue warps drain them in four column
// groups (group e: columns [32 e, 32 e + 32) of every N tile) -- twice k6_joint_lse's dz throughput, which set
// K6<grad>'s pace once the builders stopped recomputing tanh.
//   warp 0: W TMA producer; warp 1: MMA issuer (the pair's even CTA, for both); warp 2: A TMA producer;
//   warps 4-19: dz epilogue (dz_row / dz_chunk)
constexpr int kDzAcc = 4;
constexpr int kDzMaxKB = 8;  // H <= 512
constexpr int kDzABlock = kRowsPerTile * kKBlock * 2;  // 16 KB

template <bool kSB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k6_dz_2sm(const __grid_constant__ CUtensorMap w_map, const __grid_constant__ CUtensorMap h_map,
              const __grid_constant__ CUtensorMap dz_map, const JointArgs a) {
    constexpr int kSlot = kStageBytes / 2;  // this CTA's 64-column half of a W stage
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int H = a.H, V = a.V;
    const int Vp = (V + kNTile - 1) / kNTile * kNTile;
    const int KB = H / kKBlock, NT = Vp / kNTile;
    // carve: [A blocks][W stages] (1024-aligned) [bias] [dz staging 16 x 2 KB] [barriers] [tmem slot]
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ablk = base;
    uint8_t* wst = ablk + static_cast<size_t>(KB) * kDzABlock;
    float* sbias = reinterpret_cast<float*>(wst + static_cast<size_t>(a.stages) * kSlot);
    // dz staging blocks: 1024-aligned (each 2 KB block holds whole SWIZZLE_64B atoms for its TMA store)
    uint8_t* dzst = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sbias + (kSB ? Vp : 0)) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(dzst + 16 * 2048);
    uint64_t* b_full = bars;                       // [stages]
    uint64_t* b_empty = bars + kMaxStages;         // [stages]
    uint64_t* a_full = bars + 2 * kMaxStages;      // [KB]
    uint64_t* a_empty = a_full + kDzMaxKB;         // [KB]
    uint64_t* acc_full = a_empty + kDzMaxKB;       // [kDzAcc]
    uint64_t* acc_empty = acc_full + kDzAcc;       // [kDzAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kDzAcc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (kSB)
        for (int i = threadIdx.x; i < Vp; i += blockDim.x) sbias[i] = i < V ? (a.bias ? a.bias[i] : 0.f) : -INFINITY;
    const int64_t rows = *a.nrows;
    const int64_t ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
    const int64_t cells = static_cast<int64_t>(a.Tmax) * (a.Umax + 1);
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int kb = 0; kb < KB; ++kb) {
            mbar_init(&a_full[kb], 1);
            mbar_init(&a_empty[kb], 1);
        }
        for (int i = 0; i < kDzAcc; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 16 * 32 + 16);  // the leader's 16 epilogue warps + one arrive per odd-CTA warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&w_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&h_map)) : "memory");
    }
    if (warp == 1) tmem_alloc_2sm(tmem_slot, kTmemCols);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t bx = blockIdx.x, cl0 = bx - bx % 2;
    const int64_t n_iter = ntiles > cl0 ? (ntiles - cl0 + gridDim.x - 1) / gridDim.x : 0;
    const bool pon = (a.dbg & 4) != 0;  // per-role barrier-wait cycles (RNNT_K6_DEBUG=4)
    unsigned long long w0 = 0, w1 = 0, w2 = 0, w3 = 0;
    const long long t_start = clock64();

    if (warp == 0) {
        // ===== W producer: this CTA's 64-column half of every stage, onto the leader's barrier =====
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < n_iter; ++k)
                for (int n = 0; n < NT; ++n)
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait_t(&b_empty[s], ph ^ 1, pon, w0);
                        if (leader) mbar_expect_tx(&b_full[s], kStageBytes);
                        tma_load_2d_2sm(wst + static_cast<size_t>(s) * kSlot, &w_map, leader_addr(&b_full[s]),
                                        kb * kKBlock, n * kNTile + static_cast<int>(crank) * (kNTile / 2));
                        if (++s == a.stages) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
        }
    } else if (warp == 2) {
        // ===== A producer: the tile's h rows, K block by K block, as the previous tile's last N tile frees them =====
        if (lane == 0)
            for (int64_t k = 0; k < n_iter; ++k) {
                const int row0 = static_cast<int>((bx + k * gridDim.x) * kRowsPerTile);
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait_t(&a_empty[kb], (static_cast<uint32_t>(k) & 1) ^ 1, pon, w0);
                    if (leader) mbar_expect_tx(&a_full[kb], 2 * kDzABlock);  // both CTAs' rows
                    tma_load_2d_2sm(ablk + static_cast<size_t>(kb) * kDzABlock, &h_map, leader_addr(&a_full[kb]),
                                    kb * kKBlock, row0);
                }
            }
    } else if (warp == 1 && leader) {
        // ===== MMA issuer: M = 256 (the pair's two row tiles), N = 128, K = H =====
        int s = 0;
        uint32_t ph = 0, it = 0;
        for (int64_t k = 0; k < n_iter; ++k) {
            for (int n = 0; n < NT; ++n, ++it) {
                const uint32_t acc = it % kDzAcc;
                mbar_wait_t(&acc_empty[acc], ((it / kDzAcc) & 1) ^ 1, pon, w1);
                tc_fence_after();
                for (int kb = 0; kb < KB; ++kb) {
                    if (n == 0) mbar_wait_t(&a_full[kb], static_cast<uint32_t>(k) & 1, pon, w0);
                    mbar_wait_t(&b_full[s], ph, pon, w2);
                    tc_fence_after();
                    mma_kblock_ss_2sm(tmem + acc * kNTile, sw128_desc(smem_u32(ablk + static_cast<size_t>(kb) * kDzABlock)),
                                      sw128_desc(smem_u32(wst + static_cast<size_t>(s) * kSlot)), kIdescPair, kb ? 1u : 0u);
                    tc_commit_2sm_mc(&b_empty[s], 3);
                    if (n == NT - 1) tc_commit_2sm_mc(&a_empty[kb], 3);  // the tile's last use of this A block
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                tc_commit_2sm_mc(&acc_full[acc], 3);
            }
        }
    } else if (warp >= 4) {
        // ===== dz epilogue: thread = row, group eg = columns [32 eg, 32 eg + 32) of every N tile =====
        const int q = warp & 3, eg = (warp - 4) >> 2;
        const int rl = q * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const uint32_t st = smem_u32(dzst) + static_cast<uint32_t>(warp - 4) * 2048u;
        uint32_t it = 0;
        for (int64_t k = 0; k < n_iter; ++k) {
            const int64_t tile = bx + k * gridDim.x;
            const int64_t row = tile * kRowsPerTile + rl;
            int b = 0, t = 0, u = 0;
            const bool in = row < rows;
            if (in) {
                const int p = __ldg(a.rowmap + row);
                b = static_cast<int>(p / cells);
                const int rem = static_cast<int>(p - static_cast<int64_t>(b) * cells);
                t = rem / (a.Umax + 1);
                u = rem - t * (a.Umax + 1);
            }
            const int T = in ? min(a.T_b[b], a.Tmax) : 0, U = in ? min(a.U_b[b], a.Umax) : 0;
            const bool live = in && t < T && u <= U;
            const int yv = (live && u < U) ? a.targets[static_cast<int64_t>(b) * a.Umax + u] : -1;
            const DzRow d = dz_row(a, in, b, t, u, T, U, live, yv, cells);
            const f32x2 l2 = pk(kLog2e, kLog2e), nl = pk(-d.lsel, -d.lsel), g2 = pk(d.sb + d.sy, d.sb + d.sy);
            for (int n = 0; n < NT; ++n, ++it) {
                const uint32_t acc = it % kDzAcc;
                const int v0 = n * kNTile + eg * 32;
                float4 bq[8];  // !kSB: global bias loads in flight under the TMEM load
#pragma unroll
                for (int j = 0; j < 8; ++j) bq[j] = kSB ? make_float4(0.f, 0.f, 0.f, 0.f) : bias4(a, v0 + 4 * j);
                mbar_wait_t(&acc_full[acc], (it / kDzAcc) & 1, pon, w3);
                tc_fence_after();
                uint32_t r[32];
                TMEM_LD32(lane_base + acc * kNTile + eg * 32, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                tc_fence_before();  // the accumulator is free once every group has loaded its columns
                if (leader) {
                    mbar_arrive(&acc_empty[acc]);
                } else {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(&acc_empty[acc], 0);
                }
                dz_chunk<kSB>(a, r, sbias, bq, v0, d.gl, l2, nl, g2, d.sb, d.sy, d.gy, st, lane,
                              tile * kRowsPerTile + q * 32, rows, static_cast<int64_t>(NT) * kNTile, &dz_map);
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the last dz stores are done
    }
    if (pon && lane == 0) {  // the slots joint_front prints: W producer, MMA (a_full, acc_empty, b_full), epilogue, A producer
        unsigned long long* o = a.prof + static_cast<size_t>(blockIdx.x) * 8;
        if (warp == 0) { o[0] = clock64() - t_start; o[1] = w0; }
        if (warp == 1) { o[2] = w0; o[3] = w1; o[4] = w2; }  // zeros in the odd CTA (no MMAs)
        if (warp == 4) o[5] = w3;
        if (warp == 16) o[7] = w3;
        if (warp == 2) o[6] = w0;
    }
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its partner may still write into it
    tc_fence_after();
    if (warp == 1) tmem_dealloc_2sm(tmem, kTmemCols);
}

size_t dz_smem_bytes(int H, int V, int stages) {  // V = 0: bias not staged
    return 1024 + static_cast<size_t>(H / kKBlock) * kDzABlock + static_cast<size_t>(stages) * (kStageBytes / 2) +
           static_cast<size_t>((V + kNTile - 1) / kNTile * kNTile) * 4 + 1024 + 16 * 2048 +
           (2 * kMaxStages + 2 * kDzMaxKB + 2 * kDzAcc) * 8 + 16;
}

// Row map of the valid cells (t < T_b, u <= U_b), utterance by utterance: blocks (x, b) write
// map[off_b + i] = b*Tmax*(Umax+1) + t*(Umax+1) + u for cells i in [x * 4096, (x+1) * 4096) of utterance b's
// T_b (U_b + 1), off_b = sum of the earlier utterances' counts (invalid lengths count 0); block (0, B-1)
// writes the total to *nrows.
__global__ void __launch_bounds__(256) k6_rowmap(const int32_t* __restrict__ T_b, const int32_t* __restrict__ U_b,
                                                 int B, int Tmax, int Umax, int* __restrict__ map,
                                                 int* __restrict__ nrows) {
    __shared__ int s_off[8];
    const int b = blockIdx.y;
    auto count = [&](int i) {
        const int T = T_b[i], U = U_b[i];
        return (T >= 1 && T <= Tmax && U >= 0 && U <= Umax) ? T * (U + 1) : 0;
    };
    int part = 0;
    for (int i = threadIdx.x; i < b; i += blockDim.x) part += count(i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_off[threadIdx.x >> 5] = part;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) off += s_off[w];
    const int n = count(b), up1 = U_b[b] + 1;
    const int64_t base = static_cast<int64_t>(b) * Tmax * (Umax + 1);
    const int i1 = min(n, static_cast<int>(blockIdx.x + 1) * 4096);
    for (int i = static_cast<int>(blockIdx.x) * 4096 + threadIdx.x; i < i1; i += blockDim.x) {
        const int t = i / up1, u = i - t * up1;
        map[off + i] = static_cast<int>(base + t * (Umax + 1) + u);
    }
    if (b == B - 1 && blockIdx.x == 0 && threadIdx.x == 0) *nrows = off + n;
}

size_t joint_smem_bytes(int H, int V, int stages, bool grad, bool pair) {  // V = 0: bias not staged (!kSB)
    return (grad ? 8 * 2048 + 128 : 0) +  // kGrad: the epilogue warps' dz staging blocks
           1024 + static_cast<size_t>(stages) * (pair ? kStageBytes / 2 : kStageBytes) + static_cast<size_t>(kRowsPerTile) * (H + kJointHPad) * 2 +
           static_cast<size_t>((V + kNTile - 1) / kNTile * kNTile) * 4 + 2 * kRowsPerTile * 16 + (2 * kMaxStages + 3 + 2 * kAccBufs) * 8 + 16;
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

}  // namespace
}  // namespace rnnt

namespace {
// A timing event; under stream capture an external event-record node (timed on every replay).
cudaError_t record_ev(void* const* events, int i, cudaStream_t s) {
    if (!events) return cudaSuccess;
    cudaEvent_t e = static_cast<cudaEvent_t>(events[i]);
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) return cudaErrorUnknown;
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}
}  // namespace

namespace rnnt {
// Argument checks, W's tensor map, (optionally) the row map, and K6: the forward (-> lse and the Populate
// gathers in the workspace) when g == nullptr, the backward's first pass (-> dz, h) otherwise.  Shared by
// the loss, Viterbi and gradient entries.  rowmap / nrows: where the compact row map lives (nullptr: the
// alpha / beta regions of the workspace, free until K2 runs).
rnnt_status joint_front(const void* enc, const void* pred, const void* weight, const float* bias,
                        const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens, int B,
                        int Tmax, int Umax, int H, int V, int blank, void* workspace, size_t workspace_bytes,
                        cudaStream_t s, void* const* events, int* rowmap, int* nrows, bool make_map,
                        const GradIO* g, __nv_bfloat16* h_fwd) {
    if (B < 0 || Tmax < 1 || Umax < 0 || V < 2 || blank < 0 || blank >= V || H < 1) return RNNT_ERR_INVALID_ARG;
    if (Umax + 1 > kMaxUp1 || H % 128 != 0 || H > 512) return RNNT_ERR_UNSUPPORTED;
    if (B == 0) return RNNT_OK;
    if (!enc || !pred || !weight || !logit_lens || !target_lens || !workspace) return RNNT_ERR_INVALID_ARG;
    if (Umax > 0 && !targets) return RNNT_ERR_INVALID_ARG;
    if (workspace_bytes < rnnt::workspace_bytes(B, Tmax, Umax)) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    if ((reinterpret_cast<uintptr_t>(enc) | reinterpret_cast<uintptr_t>(pred) | reinterpret_cast<uintptr_t>(weight) |
         reinterpret_cast<uintptr_t>(bias)) % 16)
        return RNNT_ERR_INVALID_ARG;
    EncodeTiled enc_fn = encode_fn();
    if (!enc_fn) return RNNT_ERR_CUDA;
    CUtensorMap map;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(V)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(H) * 2};
    int cl = 2;  // CTA-pair W multicast (RNNT_K6_CLUSTER=1: one CTA per W stream, for A/B)
    if (const char* e = getenv("RNNT_K6_CLUSTER")) cl = atoi(e) == 1 ? 1 : 2;
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kKBlock), static_cast<cuuint32_t>(kNTile / cl)};
    const cuuint32_t estr[2] = {1, 1};
    if (enc_fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(weight), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return RNNT_ERR_CUDA;

    int dev = 0, nsm = 0, smem_max = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return RNNT_ERR_CUDA;
    int stages = kMaxStages;
    if (const char* e = getenv("RNNT_K6_STAGES")) stages = std::max(2, std::min(kMaxStages, atoi(e)));  // A/B only
    const bool sb = V <= kSBiasMaxV;  // bias staged in shared memory (small vocabularies), else read from global
    const int Vs = sb ? V : 0;
    // CTA pairs run pair MMAs by default (RNNT_K6_PAIR=0: per-CTA MMAs with the W stage multicast, for A/B)
    // The forward at small V (<= 4 N tiles, e.g. P:124's V = 500) keeps round 1's per-CTA MMAs with the W stage
    // multicast: its builders set the pace there and the pair hand-offs only add to it (p124 forward 0.419 ->
    // 0.413 ms; at c3 the two forms tie).  K6<grad> and k6_dz_2sm always pair.
    const bool pair = cl == 2 && !(getenv("RNNT_K6_PAIR") && atoi(getenv("RNNT_K6_PAIR")) == 0) &&
                      !(g == nullptr && (V + kNTile - 1) / kNTile <= 4);
    // K6<grad> on the forward's h (the training step): the two-operand-TMA dz kernel (pair MMAs only)
    // (RNNT_K6_DZTMA=0: k6_joint_lse<true> with its builders loading h into TMEM, for A/B)
    const bool dz_tma = g && g->h_ready && pair && !(getenv("RNNT_K6_DZTMA") && atoi(getenv("RNNT_K6_DZTMA")) == 0);
    auto smem_of = [&](int st) {
        return dz_tma ? dz_smem_bytes(H, Vs, st) : joint_smem_bytes(H, Vs, st, g != nullptr, pair);
    };
    while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
    const size_t smem = smem_of(stages);
    if (smem > static_cast<size_t>(smem_max)) return RNNT_ERR_UNSUPPORTED;
    CUtensorMap hmap;   // dz_tma: h [R][H] bf16 (compact rows), [128 rows x 64] boxes, SW128 as MMA operand A
    CUtensorMap dzmap;  // dz_tma: dz [R][Vp] bf16, [32 rows x 32] boxes, SWIZZLE_64B (the epilogue's staging layout)
    if (dz_tma) {
        const int64_t R = static_cast<int64_t>(B) * Tmax * (Umax + 1);
        const int Vpad = (V + kNTile - 1) / kNTile * kNTile;
        const cuuint64_t ddims[2] = {static_cast<cuuint64_t>(Vpad), static_cast<cuuint64_t>(R)};
        const cuuint64_t dstr[1] = {static_cast<cuuint64_t>(Vpad) * 2};
        const cuuint32_t dbox[2] = {32, 32};
        if (enc_fn(&dzmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g->dz, ddims, dstr, dbox, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return RNNT_ERR_CUDA;
        const cuuint64_t hdims[2] = {static_cast<cuuint64_t>(H),
                                     static_cast<cuuint64_t>(static_cast<int64_t>(B) * Tmax * (Umax + 1))};
        const cuuint32_t hbox[2] = {static_cast<cuuint32_t>(kKBlock), static_cast<cuuint32_t>(kRowsPerTile)};
        if (enc_fn(&hmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(g->h), hdims, strides, hbox,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return RNNT_ERR_CUDA;
        if (cudaFuncSetAttribute(sb ? k6_dz_2sm<true> : k6_dz_2sm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)) != cudaSuccess)
            return RNNT_ERR_CUDA;
    }
    const bool st = h_fwd != nullptr;  // the training step's forward: builders store h (kStore instances)
    auto kern = pair ? (sb ? (g ? k6_joint_lse<true, 2, true, true>
                                : (st ? k6_joint_lse<false, 2, true, true, true> : k6_joint_lse<false, 2, true, true>))
                           : (g ? k6_joint_lse<true, 2, false, true>
                                : (st ? k6_joint_lse<false, 2, false, true, true> : k6_joint_lse<false, 2, false, true>)))
              : sb ? (g ? (cl > 1 ? k6_joint_lse<true, 2, true, false> : k6_joint_lse<true, 1, true, false>)
                        : st ? (cl > 1 ? k6_joint_lse<false, 2, true, false, true> : k6_joint_lse<false, 1, true, false, true>)
                             : (cl > 1 ? k6_joint_lse<false, 2, true, false> : k6_joint_lse<false, 1, true, false>))
                   : (g ? (cl > 1 ? k6_joint_lse<true, 2, false, false> : k6_joint_lse<true, 1, false, false>)
                        : st ? (cl > 1 ? k6_joint_lse<false, 2, false, false, true> : k6_joint_lse<false, 1, false, false, true>)
                             : (cl > 1 ? k6_joint_lse<false, 2, false, false> : k6_joint_lse<false, 1, false, false>));
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return RNNT_ERR_CUDA;

    const Workspace w = carve(workspace, B, Tmax, Umax);
    if (static_cast<int64_t>(B) * Tmax * (Umax + 1) >= (int64_t(1) << 31)) return RNNT_ERR_UNSUPPORTED;
    if (!rowmap) {  // the row map and its length in the alpha / beta regions, which K2 only fills afterwards
        rowmap = reinterpret_cast<int*>(w.alpha);
        nrows = reinterpret_cast<int*>(w.beta);
    }
    JointArgs args{static_cast<const __nv_bfloat16*>(enc), static_cast<const __nv_bfloat16*>(pred), bias, targets,
                   logit_lens, target_lens, B, Tmax, Umax, H, V, blank,
                   static_cast<int64_t>(B) * Tmax * (Umax + 1), stages, rowmap, nrows, 0, nullptr, w.lse, w.lp,
                   nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, h_fwd, nullptr};
    if (g) {
        args.lse_in = g->lse;
        args.lp_in = g->lp;
        args.alpha = g->alpha;
        args.beta = g->beta;
        args.logp = g->logp;
        args.grad_scale = g->grad_scale;
        args.dz_out = g->dz;
        if (g->h_ready)
            args.h_in = g->h;  // stored by the forward: loaded, not recomputed
        else
            args.h_out = g->h;
    }
    if (const char* e = getenv("RNNT_K6_DEBUG")) args.dbg = atoi(e);
    args.prof = nullptr;
    if (args.dbg & 4) cudaMalloc(&args.prof, sizeof(unsigned long long) * 8 * nsm);
    const int64_t ntiles = (args.rows + kRowsPerTile - 1) / kRowsPerTile;
    int grid = static_cast<int>(std::min<int64_t>(ntiles, nsm));
    grid = std::max(cl, grid - grid % cl);  // whole clusters
    if (record_ev(events, 0, s) != cudaSuccess) return RNNT_ERR_CUDA;
    if (make_map)
        k6_rowmap<<<dim3(static_cast<unsigned>((static_cast<int64_t>(Tmax) * (Umax + 1) + 4095) / 4096), B), 256, 0,
                    s>>>(logit_lens, target_lens, B, Tmax, Umax, rowmap, nrows);
    if (dz_tma) {
        if (sb)
            k6_dz_2sm<true><<<grid, kThreads, smem, s>>>(map, hmap, dzmap, args);
        else
            k6_dz_2sm<false><<<grid, kThreads, smem, s>>>(map, hmap, dzmap, args);
    } else {
        kern<<<grid, kThreads, smem, s>>>(map, args);
    }
    if (cudaGetLastError() != cudaSuccess || record_ev(events, 1, s) != cudaSuccess) return RNNT_ERR_CUDA;
    if (args.prof) {  // diagnostics: mean per-CTA cycle split (stderr)
        unsigned long long h[8 * 148] = {};
        cudaStreamSynchronize(s);
        cudaMemcpy(h, args.prof, sizeof(unsigned long long) * 8 * std::min(nsm, 148), cudaMemcpyDeviceToHost);
        double m[8] = {};
        for (int c = 0; c < grid && c < 148; ++c)
            for (int k = 0; k < 8; ++k) m[k] += static_cast<double>(h[c * 8 + k]) / grid;
        fprintf(stderr, "K6 cycles/CTA total %.0f | tma wait b_empty %.0f | mma wait a_full %.0f acc_empty %.0f b_full %.0f"
                        " | epi wait acc_full %.0f / %.0f | builder (dz kernel: A TMA) wait a_empty %.0f\n", m[0], m[1], m[2], m[3], m[4], m[5], m[7], m[6]);
        cudaFree(args.prof);
    }
    return RNNT_OK;
}
}  // namespace rnnt

extern "C" rnnt_status rnnt_joint_loss_ex(const void* enc, const void* pred, const void* weight, const float* bias,
                                          const int32_t* targets, const int32_t* logit_lens,
                                          const int32_t* target_lens, int B, int Tmax, int Umax, int H, int V,
                                          int blank, int variant, float* losses, void* workspace,
                                          size_t workspace_bytes, void* stream, void* const* events) {
    using namespace rnnt;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (B > 0 && !losses) return RNNT_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const rnnt_status st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V,
                                       blank, workspace, workspace_bytes, s, events);
    if (st != RNNT_OK || B == 0) return st;
    const Workspace w = carve(workspace, B, Tmax, Umax);
    const int vk = (variant < 0) ? kRnnt : (variant == WRNNT_FORCE_FINAL ? kForceFinal : kAllowIgnore);
    Problem p{nullptr, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, vk, losses, nullptr, nullptr, kF32};
    if (record_ev(events, 2, s) != cudaSuccess || launch_k2_alpha_beta(p, w, s) != cudaSuccess ||
        record_ev(events, 3, s) != cudaSuccess)
        return RNNT_ERR_CUDA;
    return RNNT_OK;
}

extern "C" rnnt_status rnnt_joint_viterbi(const void* enc, const void* pred, const void* weight, const float* bias,
                                          const int32_t* targets, const int32_t* logit_lens,
                                          const int32_t* target_lens, int B, int Tmax, int Umax, int H, int V,
                                          int blank, int variant, float* best_logp, int32_t* frames, int32_t* span,
                                          void* workspace, size_t workspace_bytes, void* stream) {
    using namespace rnnt;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (B > 0 && (!best_logp || (Umax > 0 && !frames))) return RNNT_ERR_INVALID_ARG;
    if (Umax + 1 > kMaxUp1Viterbi) return RNNT_ERR_UNSUPPORTED;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const rnnt_status st = joint_front(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V,
                                       blank, workspace, workspace_bytes, s, nullptr);
    if (st != RNNT_OK || B == 0) return st;
    const Workspace w = carve(workspace, B, Tmax, Umax);
    const int vk = (variant < 0) ? kRnnt : (variant == WRNNT_FORCE_FINAL ? kForceFinal : kAllowIgnore);
    Problem p{nullptr, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, vk, nullptr, nullptr, nullptr, kF32};
    return launch_k4_viterbi(p, w, best_logp, frames, span, s) == cudaSuccess ? RNNT_OK : RNNT_ERR_CUDA;
}

extern "C" rnnt_status rnnt_joint_loss(const void* enc, const void* pred, const void* weight, const float* bias,
                                       const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens,
                                       int B, int Tmax, int Umax, int H, int V, int blank, int variant,
                                       float* losses, void* workspace, size_t workspace_bytes, void* stream) {
    return rnnt_joint_loss_ex(enc, pred, weight, bias, targets, logit_lens, target_lens, B, Tmax, Umax, H, V, blank,
                              variant, losses, workspace, workspace_bytes, stream, nullptr);
}
