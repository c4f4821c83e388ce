// k8_joint_bwd.cu -- K8 and K9: the fused joint's two backward GEMMs on the tensor cores (SURVEY §8(f) NEXT-4,
// training; readings R22, R23).  They replace the plain library GEMMs of round 1.
//
//   K8   dpre(r, :) = bf16( (sum_v dz(r, v) W(v, :)) * (1 - h(r, :)^2) )          r = a compact valid cell
//        the dh GEMM with tanh' fused into its epilogue: dh never leaves the SM in fp32 -- its only HBM trace is
//        dpre, which K7 sums over u (d enc) and t (d pred) without reading h again.
//   K9   dW(v, :) = sum_r dz(r, v) h(r, :),  dbias(v) = sum_r dz(r, v)
//        split over row ranges (K) -- the output is only V x H -- with partials reduced in a fixed order
//        (k9_reduce), so the result is deterministic.  dbias comes from the same dz tiles in shared memory.
//
// Operands (bf16, fp32 accumulation in TMEM): dz [R][Vp] and h [R][Hg] as K6 / K6<grad> write them, W [V][H] as the
// caller passes it.  K8: A = dz tile (K-major: v contiguous), B = W (MN-major: h contiguous, K = v); K9: A = dz^T
// and B = h, both MN-major (v / h contiguous, K = r).  Every operand moves by TMA as SWIZZLE_128B boxes of
// 64 elements along the contiguous dimension; the MN-major ones are read by the MMA through sw128_mn_desc.
//
// Both kernels: one CTA per SM, warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer (one elected lane),
// the rest = epilogue (and, in K9, the dbias summers).  Clusters of C CTAs share the operand that does not
// depend on the CTA's own tile: K8's W stages (C consecutive row tiles) and K9's h stages (C consecutive v
// tiles of one row range) -- each CTA fetches 1/C of the stage and multicasts it, so the L2 -> SM traffic per
// CTA is A + B / C (the bound that sets the pace of a 128-row tile against a 1 MB W).
#include <algorithm>
#include <cstdio>
#include <vector>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "joint.cuh"
#include "rnnt_b200.h"
#include "tc.cuh"

namespace rnnt {
namespace {

constexpr int kBwdMaxStages = 8;
constexpr uint32_t kBwdTmemCols = 512;

// One MMA, both operands from shared memory (descriptors), issued by one elected lane of the converged warp.
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t tmem, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols) : "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}

// K8's epilogue for one warp: its 32 rows (a TMEM lane quarter; lane 0's row = row_w) x nch chunks of 32 columns
// from column c_lo of H (TMEM columns lane_base + 32 ci): dpre = acc * (1 - h^2) in bf16.  h in and dpre out move
// as 8 whole 64-byte row segments per warp instruction through 4 KB of per-warp shared staging (h 2 KB, out
// 2 KB; 16-byte chunks XOR-swizzled by (row >> 1) & 3: conflict-free both ways); one thread per row in between.
// (Per-thread row accesses -- 32 rows x 16 B per instruction -- kept L1 ~80 % busy and set K8's pace.)
// h is fetched kPF chunks ahead, the first kPF before wait_acc() (the accumulator wait): h comes from HBM,
// and with one chunk of look-ahead its latency, not the tensor work, set K8's pace at p124 (small K).
// release() runs once this warp's last TMEM load of the accumulator has completed.
constexpr int kK8StgBytes = 4096;
constexpr int kPF = 4;
template <bool kTanh, typename Wait, typename Release>
__device__ __forceinline__ void k8_epilogue(uint32_t lane_base, int64_t row_w, int64_t R, const __nv_bfloat16* h,
                                            int Hg, __nv_bfloat16* dpre, int H, int c_lo, int nch, uint32_t stg,
                                            int lane, Wait wait_acc, Release release) {
    const uint32_t sh = stg, so = stg + 2048;
    const int sr = lane >> 2, sc = lane & 3;  // copy role: rows it * 8 + sr, 16-byte chunk sc
    auto soff = [](int row, int chunk) { return static_cast<uint32_t>(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4)); };
    uint4 hn[kPF][4];
    auto load_h = [&](int ci, uint4 (&dst)[4]) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int64_t r = row_w + it * 8 + sr;
            dst[it] = r < R ? __ldcs(reinterpret_cast<const uint4*>(h + r * Hg + c_lo + ci * 32 + sc * 8))
                            : make_uint4(0u, 0u, 0u, 0u);
        }
    };
    if constexpr (kTanh) {
#pragma unroll
        for (int ci = 0; ci < kPF; ++ci)
            if (ci < nch) load_h(ci, hn[ci]);
    }
    wait_acc();
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {  // nch <= 8 (H <= 512): unrolled so hn[] stays in registers
        if (ci >= nch) break;
        __syncwarp();
        if constexpr (kTanh) {
#pragma unroll
            for (int it = 0; it < 4; ++it) st_shared_v4(sh + soff(it * 8 + sr, sc), hn[ci % kPF][it]);
            __syncwarp();
            if (ci + kPF < nch) load_h(ci + kPF, hn[ci % kPF]);
        }
        uint32_t r[32];
        TMEM_LD32(lane_base + ci * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ci + 1 == nch) release();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t ow[4];
            if constexpr (kTanh) {
                const uint4 hq = ld_shared_v4(sh + soff(lane, i));
                const uint32_t hw[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 hh = unpack_bf16x2(hw[j]);
                    const float2 d = upk(fmul2(pk(__uint_as_float(r[8 * i + 2 * j]), __uint_as_float(r[8 * i + 2 * j + 1])),
                                              ffma2(pk(-hh.x, -hh.y), pk(hh.x, hh.y), pk(1.f, 1.f))));
                    ow[j] = pack_bf16x2(d.x, d.y);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ow[j] = pack_bf16x2(__uint_as_float(r[8 * i + 2 * j]), __uint_as_float(r[8 * i + 2 * j + 1]));
            }
            st_shared_v4(so + soff(lane, i), make_uint4(ow[0], ow[1], ow[2], ow[3]));
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int64_t r = row_w + it * 8 + sr;
            const uint4 v = ld_shared_v4(so + soff(it * 8 + sr, sc));
            if (r < R) __stcs(reinterpret_cast<uint4*>(dpre + r * H + c_lo + ci * 32 + sc * 8), v);
        }
    }
}

#define TMEM_LD16(taddr, r)                                                                                     \
    asm volatile(                                                                                               \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
        : "r"(taddr))

// The pair K8's epilogue for dh (no tanh'): the accumulator is drained FIRST -- all of this warp's 256 columns
// (or H / 2) loaded 16 at a time and packed to bf16 in 128 registers -- then released to the leader's MMA, and
// only then staged and stored (as k8_epilogue: 8 whole 64-byte row segments per instruction).  With the stores
// before the release, the next tile's MMAs waited for the whole epilogue: the single-buffered 128 x 512 fp32
// accumulator left the tensor pipe ~69 % busy (ncu); the drain itself is short (tcgen05.ld ~700 B/cycle/SM
// with 8 warps, scripts/micro/tmem_ld.cu).
template <typename Wait, typename Release>
__device__ __forceinline__ void k8_epilogue_drain(uint32_t lane_base, int64_t row_w, int64_t R, __nv_bfloat16* dh,
                                                  int H, int c_lo, int nch, uint32_t stg, int lane, Wait wait_acc,
                                                  Release release) {
    const uint32_t so = stg + 2048;
    const int sr = lane >> 2, sc = lane & 3;
    auto soff = [](int row, int chunk) { return static_cast<uint32_t>(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4)); };
    uint32_t pk16[128];  // this row's (up to) 256 columns in bf16 pairs
    wait_acc();
#pragma unroll
    for (int c16 = 0; c16 < 16; ++c16) {  // 16 loads of 16 columns (nch * 2 of them are real)
        if (c16 < 2 * nch) {
            uint32_t r[16];
            TMEM_LD16(lane_base + c16 * 16, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) pk16[c16 * 8 + j] = pack_bf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        }
    }
    release();
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {  // 32-column chunks: stage this row, store 8 rows x 64 B per instruction
        if (ci >= nch) break;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
            st_shared_v4(so + soff(lane, i), make_uint4(pk16[ci * 16 + 4 * i], pk16[ci * 16 + 4 * i + 1],
                                                         pk16[ci * 16 + 4 * i + 2], pk16[ci * 16 + 4 * i + 3]));
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int64_t r = row_w + it * 8 + sr;
            const uint4 v = ld_shared_v4(so + soff(it * 8 + sr, sc));
            if (r < R) __stcs(reinterpret_cast<uint4*>(dh + r * H + c_lo + ci * 32 + sc * 8), v);
        }
    }
}

// =============================================================================================== K8 (dh)
// A cluster of kRT x kNH CTAs: kRT consecutive 128-row tiles x kNH parts of H (<= 256 columns each).  CTA (i, j)
// (rank i * kNH + j) owns row tile i's part j: D = 128 rows x <= 256 columns, two TMEM buffers, so its epilogue
// overlaps the next tile's MMAs.  Per 64-v stage it needs dz rows [128 x 64] (shared by the kNH CTAs of row tile
// i: each fetches 128 / kNH of the rows and multicasts them to those) and W's part j [64 v x 256 h] (shared by
// the kRT CTAs of part j: each fetches 1 / kRT of its 64-column boxes and multicasts them): per CTA and stage
// 16 / kNH + 32 / kRT KB from L2 against 128 x 256 x 64 MMA work -- 16 KB per 512 MMA cycles at 2 x 4.
constexpr int kK8Threads = 384;  // warps: 0 TMA, 1 MMA, 2-3 idle, 4-11 epilogue (2 per TMEM lane quarter)
constexpr int kK8KBlock = 64;    // v per stage (one 128-byte swizzle row of the K-major A)
constexpr int kK8ABytes = 128 * kK8KBlock * 2;  // dz rows {64 v, 128 rows}
constexpr int kK8BBox = kK8KBlock * 64 * 2;     // W box {64 h, 64 v}
constexpr int kK8Part = 256;                    // H columns per CTA (one MMA's N)

struct K8Args {
    const __nv_bfloat16* h;   // [R][Hg]
    __nv_bfloat16* dpre;      // [R][H]
    int R, H, Hg, V, stages;
    bool split;               // pair kernel: the two 256-column chunks handed over separately (H = 512)
    unsigned long long* prof;  // RNNT_K8_DEBUG=4: per-CTA wait cycles [grid][8] (diagnostics), else nullptr
};

template <int kNH, int kRT>
__global__ void __cluster_dims__(kNH * kRT, 1, 1) __launch_bounds__(kK8Threads, 1)
    k8_dh_tanh(const __grid_constant__ CUtensorMap dz_map, const __grid_constant__ CUtensorMap w_map, const K8Args a) {
    constexpr int kCl = kNH * kRT;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int slot_bytes = kK8ABytes + (kK8Part / 64) * kK8BBox;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(a.stages) * slot_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kBwdMaxStages;
    uint64_t* acc_full = bars + 2 * kBwdMaxStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;             // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 4);
    const uint32_t stg0 = (smem_u32(acc_full + 6) + 127) & ~127u;  // 8 epilogue warps x kK8StgBytes
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int crank = kCl > 1 ? static_cast<int>(cluster_rank()) : 0;
    const int ti = crank / kNH, pj = crank % kNH;              // row tile in the group, part of H
    const int n0 = pj * kK8Part, width = min(kK8Part, a.H - n0);  // this CTA's H columns [n0, n0 + width)
    const int nbox = width / 64;

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCl);  // released by the MMAs of every CTA of the cluster
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dz_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&w_map)) : "memory");
    }
    if (warp == 1) tmem_alloc(tmem_slot, kBwdTmemCols);
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (static_cast<int64_t>(a.R) + 127) / 128;
    const int64_t ngroups = (ntiles + kRT - 1) / kRT, ncl = gridDim.x / kCl, cl = blockIdx.x / kCl;
    const int64_t n_iter = ngroups > cl ? (ngroups - cl + ncl - 1) / ncl : 0;  // the same for the whole cluster
    auto tile_of = [&](int64_t k) { return (cl + k * ncl) * kRT + ti; };
    const int KB = (a.V + kK8KBlock - 1) / kK8KBlock;  // dz's columns past V are zero: K stops at V
    const bool pon = a.prof != nullptr;
    unsigned long long w_empty = 0, w_full = 0, w_accempty = 0, w_accfull = 0;
    const long long t_start = clock64();

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: 1/kNH of the dz rows + 1/kRT of the W part's boxes, multicast =====
            constexpr int arows = 128 / kNH;
            const uint16_t amask = static_cast<uint16_t>(((1u << kNH) - 1) << (ti * kNH));
            uint16_t bmask = 0;
            for (int i = 0; i < kRT; ++i) bmask |= static_cast<uint16_t>(1u << (i * kNH + pj));
            int s = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < n_iter; ++k) {
                const int64_t r0 = tile_of(k) * 128;
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait_t(&empty[s], ph ^ 1, pon, w_empty);
                    mbar_expect_tx(&full[s], kK8ABytes + nbox * kK8BBox);
                    uint8_t* slot = base + static_cast<size_t>(s) * slot_bytes;
                    // rows past R (a partial or dummy tile) are zero-filled by TMA and still count their bytes
                    uint8_t* adst = slot + pj * arows * 128;
                    if constexpr (kNH > 1)
                        tma_load_2d_mc(adst, &dz_map, &full[s], kb * kK8KBlock, static_cast<int>(r0 + pj * arows), amask);
                    else
                        tma_load_2d(adst, &dz_map, &full[s], kb * kK8KBlock, static_cast<int>(r0));
                    for (int j = ti; j < nbox; j += kRT) {
                        uint8_t* dst = slot + kK8ABytes + j * kK8BBox;
                        if constexpr (kRT > 1)
                            tma_load_2d_mc(dst, &w_map, &full[s], n0 + j * 64, kb * kK8KBlock, bmask);
                        else
                            tma_load_2d(dst, &w_map, &full[s], n0 + j * 64, kb * kK8KBlock);
                    }
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: D[128 rows x width] (+)= dz[128 x 64] . W[64 x width] per stage =====
        int s = 0;
        uint32_t ph = 0;
        const uint32_t idesc = idesc_bf16(128, width, false, true);
        for (int64_t k = 0; k < n_iter; ++k) {
            const int acc = static_cast<int>(k & 1);
            mbar_wait_t(&acc_empty[acc], (static_cast<uint32_t>(k >> 1) & 1) ^ 1, pon, w_accempty);
            tc_fence_after();
            const uint32_t d_tmem = tmem + acc * kK8Part;
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait_t(&full[s], ph, pon, w_full);
                tc_fence_after();
                const uint32_t sa = smem_u32(base + static_cast<size_t>(s) * slot_bytes);
                const uint64_t adesc = sw128_desc(sa);
#pragma unroll
                for (int ks = 0; ks < kK8KBlock / 16; ++ks)
                    mma_ss(d_tmem, adesc + 2 * ks, sw128_mn_desc(sa + kK8ABytes + ks * 2048, kK8BBox), idesc,
                           (kb | ks) ? 1u : 0u);
                if constexpr (kCl > 1)
                    tc_commit_mc(&empty[s], static_cast<uint16_t>((1u << kCl) - 1));
                else
                    tc_commit(&empty[s]);
                if (++s == a.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            tc_commit(&acc_full[acc]);
        }
    } else if (warp >= 4) {
        // ===== epilogue: the two warps of a lane quarter split the part's columns (k8_epilogue) =====
        const int q = warp & 3, eh = (warp - 4) >> 2;
        const int half = width / 2, nch = half / 32;
        const int c_lo = eh * half;
        const uint32_t stg = stg0 + (warp - 4) * kK8StgBytes;
        for (int64_t k = 0; k < n_iter; ++k) {
            const int acc = static_cast<int>(k & 1);
            const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * kK8Part + c_lo;
            k8_epilogue<true>(lane_base, tile_of(k) * 128 + q * 32, a.R, a.h, a.Hg, a.dpre, a.H, n0 + c_lo, nch, stg, lane,
                        [&]() {
                            mbar_wait_t(&acc_full[acc], static_cast<uint32_t>(k >> 1) & 1, pon, w_accfull);
                            tc_fence_after();
                        },
                        [&]() {  // the last load of this buffer is done: the MMA may refill it
                            tc_fence_before();
                            mbar_arrive(&acc_empty[acc]);
                        });
        }
    }
    if (pon) {
        unsigned long long* pp = a.prof + blockIdx.x * 8;
        if (warp == 0 && lane == 0) { pp[0] = clock64() - t_start; pp[1] = w_empty; }
        if (warp == 1 && lane == 0) { pp[2] = w_full; pp[3] = w_accempty; pp[6] = n_iter; }
        if (warp == 4 && lane == 0) { pp[4] = w_accfull; pp[5] = clock64() - t_start; }
    }
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();  // no CTA leaves while a partner may still multicast into it
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, kBwdTmemCols);
}

// K8 on CTA pairs (cta_group::2): the pair's MMA has M = 256 rows (the even CTA's row tile, then the odd
// CTA's) and N = all of H in chunks of 256, each chunk's W columns split between the two CTAs -- per CTA and
// 64-v stage 16 KB of dz + H / 2 * 128 B of W = 48 KB against 256 x 512 x 64 pair MMA work (1024 cycles per
// SM): the ~47 B / cycle / SM that the chip's L2 -> SM delivery sustains (measured on K9, the same
// shape), where K8's single-CTA 128 x 256 tile needed 94.  D = 128 rows x H per CTA fills TMEM, so the
// epilogue is not double-buffered: it drains the accumulator, releases it (both CTAs' epilogue warps arrive on
// the leader's acc_empty) and finishes its last chunk while the next tile's MMAs start.
template <int NC>
__device__ __forceinline__ void mma_stage_k8_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t id0, uint32_t id1,
                                                 uint32_t accumulate) {
    // 4 K steps of 16 v: A (K-major) +32 B (desc +2), B (MN-major) +2048 B (desc +128); chunk 1: D + 256
    // columns, B + 2 boxes of 8 KB (desc +1024)
    if constexpr (NC == 1) {
        asm volatile(
            "{\n"
            ".reg .pred p, q, e;\n"
            ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "setp.eq.b32 q, %4, %4;\n"
            "add.u64 a1, %1, 2;\n add.u64 a2, %1, 4;\n add.u64 a3, %1, 6;\n"
            "add.u64 b1, %2, 128;\n add.u64 b2, %2, 256;\n add.u64 b3, %2, 384;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
            "}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id0), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n"
            ".reg .pred p, q, e;\n"
            ".reg .b32 d1;\n"
            ".reg .b64 a1, a2, a3, b1, b2, b3, c0, c1, c2, c3;\n"
            "setp.ne.b32 p, %5, 0;\n"
            "setp.eq.b32 q, %5, %5;\n"
            "add.u32 d1, %0, 256;\n"
            "add.u64 a1, %1, 2;\n add.u64 a2, %1, 4;\n add.u64 a3, %1, 6;\n"
            "add.u64 b1, %2, 128;\n add.u64 b2, %2, 256;\n add.u64 b3, %2, 384;\n"
            "add.u64 c0, %2, 1024;\n add.u64 c1, b1, 1024;\n add.u64 c2, b2, 1024;\n add.u64 c3, b3, 1024;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], %1, c0, %4, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a1, c1, %4, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a2, c2, %4, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a3, c3, %4, q;\n"
            "}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id0), "r"(id1), "r"(accumulate)
            : "memory");
    }
}

template <bool kTanh>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kK8Threads, 1)
    k8_dh_tanh_2sm(const __grid_constant__ CUtensorMap dz_map, const __grid_constant__ CUtensorMap w_map, const K8Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int H = a.H;
    const int nb = H / 128;  // W boxes {64 h, 64 v} per CTA and stage (half of each 256-column chunk)
    const int slot_bytes = kK8ABytes + nb * kK8BBox;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(a.stages) * slot_bytes);
    uint64_t* full = bars;                    // [stages], the leader's counts
    uint64_t* empty = bars + kBwdMaxStages;   // [stages]
    // acc_full / acc_empty [2]: with H > 256 the accumulator's two 256-column chunks are handed over separately --
    // the last stage of a tile finishes chunk 0 first, its epilogue group drains it while chunk 1's MMAs run, and
    // the next tile's first stage starts chunk 0 once that half is free (RNNT_K8_SPLIT=0: one hand-over, A/B)
    uint64_t* acc_full = bars + 2 * kBwdMaxStages;
    uint64_t* acc_empty = acc_full + 2;       // the leader's counts both CTAs' epilogue warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 4);
    const uint32_t stg0 = (smem_u32(acc_full + 6) + 127) & ~127u;  // 8 epilogue warps x kK8StgBytes
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_rank());
    const bool leader = rank == 0;
    const bool split = a.split && H == 512;  // the epilogue groups' halves are the two chunks only at H = 512

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], split ? 8 : 16);  // per chunk: its 4 warps in each CTA; else all 8 in each
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dz_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&w_map)) : "memory");
    }
    if (warp == 1) tmem_alloc_2sm(tmem_slot, kBwdTmemCols);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t ntiles = (static_cast<int64_t>(a.R) + 255) / 256;
    const int64_t np = gridDim.x / 2, pr = blockIdx.x / 2;
    const int64_t n_iter = ntiles > pr ? (ntiles - pr + np - 1) / np : 0;
    const int KB = (a.V + kK8KBlock - 1) / kK8KBlock;  // dz's columns past V are zero: K stops at V
    const bool pon = a.prof != nullptr;
    unsigned long long w_empty = 0, w_full = 0, w_accempty = 0, w_accfull = 0;
    const long long t_start = clock64();

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer (both CTAs): own 128 dz rows + own half of W's columns =====
            int s = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < n_iter; ++k) {
                const int64_t r0 = (pr + k * np) * 256 + rank * 128;
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait_t(&empty[s], ph ^ 1, pon, w_empty);
                    if (leader) mbar_expect_tx(&full[s], 2 * slot_bytes);
                    uint8_t* slot = base + static_cast<size_t>(s) * slot_bytes;
                    const uint32_t lbar = leader_addr(&full[s]);
                    // rows past R (a partial or dummy tile) are zero-filled by TMA and still count their bytes
                    tma_load_2d_2sm(slot, &dz_map, lbar, kb * kK8KBlock, static_cast<int>(r0));
                    for (int n0 = 0, j = 0; n0 < H; n0 += 256) {
                        const int half = min(256, H - n0) / 2;
                        for (int c = 0; c < half; c += 64, ++j)
                            tma_load_2d_2sm(slot + kK8ABytes + j * kK8BBox, &w_map, lbar, n0 + rank * half + c,
                                            kb * kK8KBlock);
                    }
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // ===== pair MMA issuer: D[256 rows x H] (+)= dz[256 x 64] . W[64 x H] per stage =====
            int s = 0;
            uint32_t ph = 0;
            const uint32_t id0 = idesc_bf16(256, min(256, H), false, true);
            const uint32_t id1 = H > 256 ? idesc_bf16(256, H - 256, false, true) : 0u;
            for (int64_t k = 0; k < n_iter; ++k) {
                const uint32_t pe = (static_cast<uint32_t>(k) & 1) ^ 1;
                if (!split) {
                    mbar_wait_t(&acc_empty[0], pe, pon, w_accempty);
                    tc_fence_after();
                }
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait_t(&full[s], ph, pon, w_full);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(base + static_cast<size_t>(s) * slot_bytes);
                    const uint64_t adesc = sw128_desc(sa), bdesc = sw128_mn_desc(sa + kK8ABytes, kK8BBox);
                    if (split && (kb == 0 || kb == KB - 1)) {  // the chunks one after the other, each handed over
                        // chunk 1 = D + 256 columns, B + 2 boxes of 8 KB (descriptor + 1024)
                        if (kb == 0) {
                            mbar_wait_t(&acc_empty[0], pe, pon, w_accempty);
                            tc_fence_after();
                        }
                        mma_stage_k8_2sm<1>(tmem, adesc, bdesc, id0, 0u, kb ? 1u : 0u);
                        if (kb == KB - 1) tc_commit_2sm_mc(&acc_full[0], 3);
                        if (kb == 0) {
                            mbar_wait_t(&acc_empty[1], pe, pon, w_accempty);
                            tc_fence_after();
                        }
                        mma_stage_k8_2sm<1>(tmem + 256, adesc, bdesc + 1024, id1, 0u, kb ? 1u : 0u);
                        if (kb == KB - 1) tc_commit_2sm_mc(&acc_full[1], 3);
                    } else if (H > 256) {
                        mma_stage_k8_2sm<2>(tmem, adesc, bdesc, id0, id1, kb ? 1u : 0u);
                    } else {
                        mma_stage_k8_2sm<1>(tmem, adesc, bdesc, id0, 0u, kb ? 1u : 0u);
                    }
                    tc_commit_2sm_mc(&empty[s], 3);
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (!split) tc_commit_2sm_mc(&acc_full[0], 3);
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue (both CTAs): the two warps of a lane quarter split H (k8_epilogue) =====
        const int q = warp & 3, eh = (warp - 4) >> 2;
        const int half = H / 2, nch = half / 32;
        const int c_lo = eh * half;
        const uint32_t stg = stg0 + (warp - 4) * kK8StgBytes;
        for (int64_t k = 0; k < n_iter; ++k) {
            const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + c_lo;
            const int hc = split ? eh : 0;  // this group's chunk barrier
            auto wait = [&]() {
                mbar_wait_t(&acc_full[hc], static_cast<uint32_t>(k) & 1, pon, w_accfull);
                tc_fence_after();
            };
            auto release = [&]() {  // this warp's last load of the accumulator: release it to the leader
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader)
                        mbar_arrive(&acc_empty[hc]);
                    else
                        mbar_arrive_remote(&acc_empty[hc], 0);
                }
            };
            const int64_t row_w = (pr + k * np) * 256 + rank * 128 + q * 32;
            if constexpr (kTanh)
                k8_epilogue<true>(lane_base, row_w, a.R, a.h, a.Hg, a.dpre, H, c_lo, nch, stg, lane, wait, release);
            else
                k8_epilogue_drain(lane_base, row_w, a.R, a.dpre, H, c_lo, nch, stg, lane, wait, release);
        }
    }
    if (pon) {
        unsigned long long* pp = a.prof + blockIdx.x * 8;
        if (warp == 0 && lane == 0) { pp[0] = clock64() - t_start; pp[1] = w_empty; }
        if (warp == 1 && lane == 0) { pp[2] = w_full; pp[3] = w_accempty; pp[6] = n_iter; }
        if (warp == 4 && lane == 0) { pp[4] = w_accfull; pp[5] = clock64() - t_start; }
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_2sm(tmem, kBwdTmemCols);
}

// =============================================================================================== K9 (dW)
constexpr int kK9Threads = 384;  // warps: 0 TMA, 1 MMA, 2-3 idle, 4-7 dbias summers, 8-11 epilogue
constexpr int kK9Rows = 64;      // K (rows) per stage: ~1100 MMA cycles, well above a stage's ~200-cycle
                                 // barrier round trip (scripts/micro/pipe_rate.cu); 32 rows left K9 issue-bound
constexpr int kK9Box = 64 * kK9Rows * 2;  // one {64 elements, 64 rows} box, 8 KB
constexpr int kK9MaxCtas = 256;

struct K9Args {
    float* part;    // [splits][Vp][H] fp32 partial dW
    float* part_b;  // [splits][Vp] partial dbias
    int R, H, Vp, nvt, groups, splits, stages_per_split, stages;
    int dbg;  // timing ablations (env RNNT_K9_DEBUG, wrong results): 1 = no MMAs, 2 = no TMA loads;
              // 4 = per-role wait cycles (correct results) into prof, printed to stderr
    unsigned long long* prof;  // [gridDim.x][8]
};

// dbias helper for K9: thread t (of 128) sums the 16-byte chunk (t & 7) of box ((t >> 3) & 1) -- v = box * 64 +
// (t & 7) * 8 + e, e < 8 -- over rows k = (t >> 4) + 8 i of a kK9Rows-row MN-major SWIZZLE_128B dz^T stage
// (row k, chunk j at k * 128 + ((j ^ (k & 7)) << 4) in its box): kK9Rows / 8 16-byte shared loads per stage.
__device__ __forceinline__ void dbias_stage(uint32_t stage_addr, int t, float (&acc)[8]) {
    const int j = t & 7, box = (t >> 3) & 1, rg = t >> 4;
#pragma unroll
    for (int i = 0; i < kK9Rows / 8; ++i) {
        const int k = rg + 8 * i;
        uint32_t w0, w1, w2, w3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                     : "r"(stage_addr + box * kK9Box + k * 128 + ((j ^ (k & 7)) << 4)));
        const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = unpack_bf16x2(w[e]);
            acc[2 * e] += f.x;
            acc[2 * e + 1] += f.y;
        }
    }
}
// Combine the 8 row groups' partials (through shared memory `red`, 8 x 128 floats) in a fixed order; returns the
// column sum of v = t for thread t < 128.  All 128 dbias threads call it (named barrier 1).
__device__ __forceinline__ float dbias_combine(float* red, int t, const float (&acc)[8]) {
    const int j = t & 7, box = (t >> 3) & 1, rg = t >> 4;
#pragma unroll
    for (int e = 0; e < 8; ++e) red[rg * 128 + box * 64 + j * 8 + e] = acc[e];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    float o = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) o += red[g * 128 + t];
    return o;
}

template <int kCl>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kK9Threads, 1)
    k9_dw(const __grid_constant__ CUtensorMap dz_map, const __grid_constant__ CUtensorMap h_map, const K9Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int H = a.H, nbox = H / 64;
    const int slot_bytes = (2 + nbox) * kK9Box;  // A: dz^T {128 v} as 2 boxes; B: h {H} as H / 64 boxes
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(a.stages) * slot_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kBwdMaxStages;
    uint64_t* acc_full = bars + 2 * kBwdMaxStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
    float* red = reinterpret_cast<float*>(acc_full + 2);  // [8][128] dbias row-group partials
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // work unit: blockIdx.x = (split * groups + group) * kCl + rank; v tile = group * kCl + rank
    const int cl = blockIdx.x / kCl, crank = kCl > 1 ? static_cast<int>(cluster_rank()) : 0;
    const int split = cl / a.groups, vt = (cl % a.groups) * kCl + crank;
    const int64_t nst_total = (static_cast<int64_t>(a.R) + kK9Rows - 1) / kK9Rows;
    const int64_t st0 = static_cast<int64_t>(split) * a.stages_per_split;
    const int nst = static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(a.stages_per_split, nst_total - st0)));
    const int v0 = vt * 128;

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCl + 4);  // every CTA's MMAs (multicast commit) + this CTA's 4 dbias warps
        }
        mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dz_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&h_map)) : "memory");
    }
    if (warp == 1) tmem_alloc(tmem_slot, kBwdTmemCols);
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: own dz^T boxes + 1/kCl of the h boxes, multicast =====
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nst; ++i) {
                const int r = static_cast<int>((st0 + i) * kK9Rows);
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], slot_bytes - (vt < a.nvt ? 0 : 2 * kK9Box));
                uint8_t* slot = base + static_cast<size_t>(s) * slot_bytes;
                if (vt < a.nvt) {  // a dummy v tile (the cluster's lockstep) loads no A
                    tma_load_2d(slot, &dz_map, &full[s], v0, r);
                    tma_load_2d(slot + kK9Box, &dz_map, &full[s], v0 + 64, r);
                }
                for (int j = crank; j < nbox; j += kCl) {
                    if constexpr (kCl > 1)
                        tma_load_2d_mc(slot + (2 + j) * kK9Box, &h_map, &full[s], j * 64, r,
                                       static_cast<uint16_t>((1u << kCl) - 1));
                    else
                        tma_load_2d(slot + (2 + j) * kK9Box, &h_map, &full[s], j * 64, r);
                }
                if (++s == a.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: D[128 v x H] (+)= dz^T[128 v x 32 r] . h[32 r x H] per stage =====
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nst; ++i) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(base + static_cast<size_t>(s) * slot_bytes);
#pragma unroll
            for (int ks = 0; ks < kK9Rows / 16; ++ks) {
                const uint64_t adesc = sw128_mn_desc(sa + ks * 2048, kK9Box);
                for (int n0 = 0; n0 < H; n0 += 256) {
                    const int N = min(256, H - n0);
                    const uint64_t bdesc = sw128_mn_desc(sa + (2 + n0 / 64) * kK9Box + ks * 2048, kK9Box);
                    mma_ss(tmem + n0, adesc, bdesc, idesc_bf16(128, N, true, true), (i | ks) ? 1u : 0u);
                }
            }
            if constexpr (kCl > 1)
                tc_commit_mc(&empty[s], static_cast<uint16_t>((1u << kCl) - 1));
            else
                tc_commit(&empty[s]);
            if (++s == a.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        tc_commit(acc_full);
    } else if (warp >= 4 && warp < 8) {
        // ===== dbias: thread = v (128 of the tile), sums its column of every dz^T stage from shared memory =====
        const int vl = threadIdx.x - 128;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nst; ++i) {
            mbar_wait(&full[s], ph);
            dbias_stage(smem_u32(base + static_cast<size_t>(s) * slot_bytes), vl, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        const float o = dbias_combine(red, vl, acc);
        if (vt < a.nvt) a.part_b[static_cast<int64_t>(split) * a.Vp + v0 + vl] = o;
    } else if (warp >= 8) {
        // ===== epilogue: thread = v (TMEM lane), the row range's partial dW for its v, all H columns =====
        const int q = warp & 3;
        const int vl = q * 32 + lane;
        mbar_wait(acc_full, 0);
        tc_fence_after();
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        float* out = a.part + (static_cast<int64_t>(split) * a.Vp + v0 + vl) * H;
        for (int c0 = 0; c0 < H; c0 += 32) {
            uint32_t r[32];
            TMEM_LD32(lane_base + c0, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (vt < a.nvt) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float4 o = nst > 0 ? make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                     __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);  // an empty row range: no MMA ran
                    reinterpret_cast<float4*>(out + c0)[i] = o;
                }
            }
        }
    }
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, kBwdTmemCols);
}

// One K9 pair stage: kK9Rows / 16 = 4 K steps x NC N chunks of pair MMAs in ONE asm block with one election
// (per-MMA asm statements re-elect and move both descriptors into uniform registers each time: issuing a
// 256 x 256 x 16 MMA took ~180 cycles against its 128 of tensor work, and the issue rate set K9's pace).
// K step: +2048 B on both MN-major descriptors (start field +128); N chunk 1: D + 256 columns, B + 2 boxes.
template <int NC>
__device__ __forceinline__ void mma_stage_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t id0, uint32_t id1,
                                              uint32_t accumulate) {
    static_assert(kK9Rows == 64, "4 K steps per stage");
    constexpr uint64_t kBox1 = (2 * kK9Box) >> 4;
    if constexpr (NC == 1) {
        asm volatile(
            "{\n"
            ".reg .pred p, q, e;\n"
            ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "setp.eq.b32 q, %4, %4;\n"
            "add.u64 a1, %1, 128;\n add.u64 a2, %1, 256;\n add.u64 a3, %1, 384;\n"
            "add.u64 b1, %2, 128;\n add.u64 b2, %2, 256;\n add.u64 b3, %2, 384;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
            "}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id0), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n"
            ".reg .pred p, q, e;\n"
            ".reg .b32 d1;\n"
            ".reg .b64 a1, a2, a3, b1, b2, b3, c0, c1, c2, c3;\n"
            "setp.ne.b32 p, %5, 0;\n"
            "setp.eq.b32 q, %5, %5;\n"
            "add.u32 d1, %0, 256;\n"
            "add.u64 a1, %1, 128;\n add.u64 a2, %1, 256;\n add.u64 a3, %1, 384;\n"
            "add.u64 b1, %2, 128;\n add.u64 b2, %2, 256;\n add.u64 b3, %2, 384;\n"
            "add.u64 c0, %2, %6;\n add.u64 c1, b1, %6;\n add.u64 c2, b2, %6;\n add.u64 c3, b3, %6;\n"
            "elect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], %1, c0, %4, p;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a1, c1, %4, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a2, c2, %4, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, q;\n"
            "@e tcgen05.mma.cta_group::2.kind::f16 [d1], a3, c3, %4, q;\n"
            "}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id0), "r"(id1), "r"(accumulate), "l"(kBox1)
            : "memory");
    }
}

// K9 on CTA pairs (cta_group::2): the pair's MMA has M = 256 (v0 .. v0 + 255: the even CTA's dz^T rows
// [v0, v0 + 128), the odd CTA's [v0 + 128, v0 + 256)) and each N = 256 chunk of H split between them (the even CTA
// holds columns [n0, n0 + N/2), the odd [n0 + N/2, n0 + N)), so per CTA and 32-row stage the shared memory fills
// with 8 KB of dz^T + H / 2 * 64 B of h = 16 KB at H = 512 against 4 x (128 x 256 x 16) MMA work -- 2.5x less
// than K9's single-CTA 128 x 512 tile (40 KB), whose fill rate set its pace (~36 B / cycle / SM measured; the
// chip's L2 -> SM delivery, not multicast, is the limit).  Only the even CTA issues MMAs; both CTAs' loads
// (2-SM TMA) complete on its full barrier, armed with the pair's bytes by its producer.  The MMA completion
// is multicast to both CTAs' mma_done barrier; each CTA's dbias warps wait on that (the stage has landed and
// been consumed), sum their dz^T columns, and free the stage (empty) for that CTA's producer.  (A relayed
// arrive from the odd CTA's dbias warps to the leader cost a MEMBAR.ALL.GPU per stage: 2.4x slower.)
template <int kDummy>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kK9Threads, 1)
    k9_dw_2sm(const __grid_constant__ CUtensorMap dz_map, const __grid_constant__ CUtensorMap h_map, const K9Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int H = a.H;
    const int hb = H / 128;                         // h boxes per CTA and stage (half of H / 64)
    const int slot_bytes = (2 + hb) * kK9Box;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(a.stages) * slot_bytes);
    uint64_t* full = bars;                        // [stages] (the leader's is the one that counts)
    uint64_t* empty = bars + kBwdMaxStages;       // [stages]
    uint64_t* mma_done = bars + 2 * kBwdMaxStages;  // [stages]
    uint64_t* acc_full = bars + 3 * kBwdMaxStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
    float* red = reinterpret_cast<float*>(acc_full + 2);  // [8][128] dbias row-group partials
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_rank());
    const bool leader = rank == 0;
    // work unit: blockIdx.x = (split * groups + group) * 2 + rank; group = a pair's 256 v
    const int cl = blockIdx.x >> 1;
    const int split = cl / a.groups, g = cl % a.groups;
    const int vt = g * 2 + rank;  // this CTA's 128-v tile
    const bool a_in = vt < a.nvt;
    const int pair_abytes = ((g * 2 < a.nvt) + (g * 2 + 1 < a.nvt)) * 2 * kK9Box;  // both CTAs' dz^T bytes
    const int64_t nst_total = (static_cast<int64_t>(a.R) + kK9Rows - 1) / kK9Rows;
    const int64_t st0 = static_cast<int64_t>(split) * a.stages_per_split;
    const int nst = static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(a.stages_per_split, nst_total - st0)));
    const int v0 = vt * 128;

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);      // the leader's producer (with the pair's bytes)
            mbar_init(&mma_done[s], 1);  // the pair MMA's multicast commit
            mbar_init(&empty[s], 4);     // this CTA's 4 dbias warps, after mma_done
        }
        mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dz_map)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&h_map)) : "memory");
    }
    if (warp == 1) tmem_alloc_2sm(tmem_slot, kBwdTmemCols);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const bool pon = (a.dbg & 4) != 0;
    unsigned long long w0 = 0, w1 = 0, w2 = 0;
    const long long t_start = clock64();

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer (both CTAs): own dz^T boxes + own h columns, on the leader's barrier =====
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nst; ++i) {
                const int r = static_cast<int>((st0 + i) * kK9Rows);
                mbar_wait_t(&empty[s], ph ^ 1, pon, w0);
                if (leader) mbar_expect_tx(&full[s], (a.dbg & 2) ? 0 : pair_abytes + 2 * hb * kK9Box);
                uint8_t* slot = base + static_cast<size_t>(s) * slot_bytes;
                const uint32_t lbar = leader_addr(&full[s]);
                if (a.dbg & 2) {
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                    continue;
                }
                if (a_in) {
                    tma_load_2d_2sm(slot, &dz_map, lbar, v0, r);
                    tma_load_2d_2sm(slot + kK9Box, &dz_map, lbar, v0 + 64, r);
                }
                for (int n0 = 0, j = 0; n0 < H; n0 += 256) {
                    const int N = min(256, H - n0), half = N / 2;
                    for (int c = 0; c < half; c += 64, ++j)
                        tma_load_2d_2sm(slot + (2 + j) * kK9Box, &h_map, lbar, n0 + rank * half + c, r);
                }
                if (++s == a.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // ===== pair MMA issuer: D[256 v x H] (+)= dz^T[256 v x 32 r] . h[32 r x H] per stage =====
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nst; ++i) {
                mbar_wait_t(&full[s], ph, pon, w1);
                tc_fence_after();
                const uint32_t sa = smem_u32(base + static_cast<size_t>(s) * slot_bytes);
                const uint64_t adesc = sw128_mn_desc(sa, kK9Box);
                const uint64_t bdesc = sw128_mn_desc(sa + 2 * kK9Box, kK9Box);
                if (!(a.dbg & 1)) {
                    if (H > 256)
                        mma_stage_2sm<2>(tmem, adesc, bdesc, idesc_bf16(256, 256, true, true),
                                         idesc_bf16(256, H - 256, true, true), i ? 1u : 0u);
                    else
                        mma_stage_2sm<1>(tmem, adesc, bdesc, idesc_bf16(256, H, true, true), 0u, i ? 1u : 0u);
                }
                tc_commit_2sm_mc(&mma_done[s], 3);
                if (++s == a.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            tc_commit_2sm_mc(acc_full, 3);
        }
    } else if (warp >= 4 && warp < 8) {
        // ===== dbias: thread = v (128 of this CTA's tile), sums its column of every dz^T stage from shared
        // memory once the pair MMA has consumed it, then frees the stage =====
        const int vl = threadIdx.x - 128;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nst; ++i) {
            mbar_wait_t(&mma_done[s], ph, pon, w2);
            dbias_stage(smem_u32(base + static_cast<size_t>(s) * slot_bytes), vl, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        const float o = dbias_combine(red, vl, acc);
        if (a_in) a.part_b[static_cast<int64_t>(split) * a.Vp + v0 + vl] = o;
    } else if (warp >= 8) {
        // ===== epilogue (both CTAs): thread = v (TMEM lane), the row range's partial dW, all H columns =====
        const int q = warp & 3;
        const int vl = q * 32 + lane;
        mbar_wait(acc_full, 0);
        tc_fence_after();
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        float* out = a.part + (static_cast<int64_t>(split) * a.Vp + v0 + vl) * H;
        for (int c0 = 0; c0 < H; c0 += 32) {
            uint32_t r[32];
            TMEM_LD32(lane_base + c0, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (a_in) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float4 o = nst > 0 ? make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                     __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);  // an empty row range: no MMA ran
                    reinterpret_cast<float4*>(out + c0)[i] = o;
                }
            }
        }
    }
    if (pon) {
        unsigned long long* pr = a.prof + blockIdx.x * 8;
        if (warp == 0 && lane == 0) { pr[0] = clock64() - t_start; pr[1] = w0; }
        if (warp == 1 && lane == 0 && leader) pr[2] = w1;
        if (warp == 4 && lane == 0) pr[3] = w2;
        if (warp == 8 && lane == 0) pr[4] = clock64() - t_start;
        if (warp == 0 && lane == 0) pr[5] = nst;
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_2sm(tmem, kBwdTmemCols);
}

// dW(v, :) = sum over splits (in order) of the partials, dbias(v) likewise; v < V only.
__global__ void __launch_bounds__(256) k9_reduce(const float* __restrict__ part, const float* __restrict__ part_b,
                                                 int splits, int V, int Vp, int H, float* __restrict__ dw,
                                                 float* __restrict__ db) {
    const int64_t n4 = static_cast<int64_t>(V) * H / 4;
    const int64_t stride4 = static_cast<int64_t>(Vp) * H / 4;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4 + V;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < n4) {
            // split order kept (deterministic); eight loads in flight before their adds, which were a chain of
            // dependent global loads otherwise (12 us at p124 for 19 MB)
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            int s = 0;
            for (; s + 8 <= splits; s += 8) {
                float4 p[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) p[k] = __ldcs(p4 + (s + k) * stride4 + i);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    o.x += p[k].x;
                    o.y += p[k].y;
                    o.z += p[k].z;
                    o.w += p[k].w;
                }
            }
            for (; s < splits; ++s) {
                const float4 p = __ldcs(p4 + s * stride4 + i);
                o.x += p.x;
                o.y += p.y;
                o.z += p.z;
                o.w += p.w;
            }
            reinterpret_cast<float4*>(dw)[i] = o;
        } else if (db) {
            const int v = static_cast<int>(i - n4);
            float o = 0.f;
            for (int s = 0; s < splits; ++s) o += part_b[static_cast<int64_t>(s) * Vp + v];
            db[v] = o;
        }
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D bf16 tensor map: inner dimension d0 (contiguous, row pitch `pitch` elements), outer d1; box {b0, b1};
// SWIZZLE_128B; out-of-bounds boxes are zero-filled.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t pitch, uint32_t b0, uint32_t b1) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return false;
    const cuuint64_t dims[2] = {d0, d1};
    const cuuint64_t strides[1] = {pitch * 2};
    const cuuint32_t box[2] = {b0, b1};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count_and_smem(int* smem_max) {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return 0;
    return nsm;
}

// How many clusters of `cl` CTAs with `smem` bytes each can be resident at once (a cluster must fit in one GPC:
// with one CTA per SM, fewer than nsm / cl for cl > 2).  0 on error.
template <typename K>
int max_clusters(K kern, int cl, size_t smem, int threads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Largest cluster size <= cap that divides n (a power of two).
int cluster_for(int n, int cap) {
    int c = 1;
    while (c * 2 <= cap && n % (c * 2) == 0) c *= 2;
    return c;
}

}  // namespace

// K9's partials: splits * Vp <= max(number of CTAs, nvt) * 128 rows of H + 1 floats; CTAs <= kK9MaxCtas.
size_t k9_partial_bytes(int Vp, int H) {
    const size_t rows = std::max<size_t>(static_cast<size_t>(kK9MaxCtas) * 128, static_cast<size_t>(Vp));
    return sizeof(float) * rows * (static_cast<size_t>(H) + 1);
}

cudaError_t launch_k8(const __nv_bfloat16* dz, const __nv_bfloat16* weight, const __nv_bfloat16* h,
                      __nv_bfloat16* dpre, int R, int H, int Hg, int V, int Vp, bool tanh_in_k8, cudaStream_t s) {
    if (R <= 0) return cudaSuccess;
    int smem_max = 0;
    const int nsm = sm_count_and_smem(&smem_max);
    if (!nsm) return cudaErrorUnknown;
    if (!getenv("RNNT_K8_RT")) {  // default: CTA pairs (cta_group::2); RNNT_K8_RT=n: the 2-D cluster kernel (A/B)
        CUtensorMap dz_map, w_map;
        if (!make_map(&dz_map, dz, Vp, R, Vp, kK8KBlock, 128) || !make_map(&w_map, weight, H, V, H, 64, kK8KBlock))
            return cudaErrorUnknown;
        const int slot = kK8ABytes + (H / 128) * kK8BBox;
        int stages = kBwdMaxStages;
        auto smem_of = [&](int st) {
            return static_cast<size_t>(1024 + st * slot + (2 * kBwdMaxStages + 6) * 8 + 128 + 8 * kK8StgBytes);
        };
        while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
        const size_t smem = smem_of(stages);
        auto kern2 = tanh_in_k8 ? k8_dh_tanh_2sm<true> : k8_dh_tanh_2sm<false>;
        if (cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
            return cudaErrorInvalidConfiguration;
        const int64_t ntiles = (static_cast<int64_t>(R) + 255) / 256;
        int resident = max_clusters(kern2, 2, smem, kK8Threads);
        if (resident <= 0) resident = nsm / 2;
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, resident))) * 2;
        const bool split = !(getenv("RNNT_K8_SPLIT") && atoi(getenv("RNNT_K8_SPLIT")) == 0);
        K8Args args{h, dpre, R, H, Hg, V, stages, split, nullptr};
        const bool prof = getenv("RNNT_K8_DEBUG") && (atoi(getenv("RNNT_K8_DEBUG")) & 4);
        if (prof) cudaMalloc(&args.prof, sizeof(unsigned long long) * 8 * grid);
        kern2<<<grid, kK8Threads, smem, s>>>(dz_map, w_map, args);
        if (cudaGetLastError() != cudaSuccess) return cudaErrorUnknown;
        if (prof) {
            std::vector<unsigned long long> hh(8 * grid);
            cudaStreamSynchronize(s);
            cudaMemcpy(hh.data(), args.prof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost);
            double m[8] = {};
            for (int c = 0; c < grid; ++c)
                for (int k = 0; k < 8; ++k) m[k] += static_cast<double>(hh[c * 8 + k]) / grid;
            fprintf(stderr, "K8 pair grid %d stages %d | cycles/CTA %.0f | producer wait empty %.0f | MMA wait full %.0f, "
                            "acc_empty %.0f (x2: leaders only) | epilogue wait acc_full %.0f, end %.0f | tiles/CTA %.0f\n",
                    grid, stages, m[0], m[1], 2 * m[2], 2 * m[3], m[4], m[5], m[6]);
            cudaFree(args.prof);
        }
        return cudaGetLastError();
    }
    const int nh = (H + kK8Part - 1) / kK8Part;  // parts of H: 1 (H <= 256) or 2
    int rt = 4;  // row tiles per cluster (W multicast), 2 x 4 or 1 x 4 CTAs
    if (const char* e = getenv("RNNT_K8_RT")) rt = atoi(e) >= 4 ? 4 : atoi(e) >= 2 ? 2 : 1;
    CUtensorMap dz_map, w_map;
    if (!make_map(&dz_map, dz, Vp, R, Vp, kK8KBlock, 128 / nh) || !make_map(&w_map, weight, H, V, H, 64, kK8KBlock))
        return cudaErrorUnknown;
    constexpr int slot = kK8ABytes + (kK8Part / 64) * kK8BBox;
    int stages = kBwdMaxStages;
    auto smem_of = [&](int st) {
        return static_cast<size_t>(1024 + st * slot + (2 * kBwdMaxStages + 6) * 8 + 128 + 8 * kK8StgBytes);
    };
    while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
    const size_t smem = smem_of(stages);
    if (smem > static_cast<size_t>(smem_max)) return cudaErrorInvalidConfiguration;
    auto kern = nh == 2 ? (rt == 4 ? k8_dh_tanh<2, 4> : rt == 2 ? k8_dh_tanh<2, 2> : k8_dh_tanh<2, 1>)
                        : (rt == 4 ? k8_dh_tanh<1, 4> : rt == 2 ? k8_dh_tanh<1, 2> : k8_dh_tanh<1, 1>);
    const int cl = nh * rt;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return cudaErrorInvalidConfiguration;
    const int64_t ngroups = ((static_cast<int64_t>(R) + 127) / 128 + rt - 1) / rt;
    int resident = max_clusters(kern, cl, smem, kK8Threads);  // persistent: only co-resident clusters
    if (resident <= 0) resident = nsm / cl;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ngroups, resident))) * cl;
    K8Args args{h, dpre, R, H, Hg, V, stages, false, nullptr};
    const bool prof = getenv("RNNT_K8_DEBUG") && (atoi(getenv("RNNT_K8_DEBUG")) & 4);
    if (prof) cudaMalloc(&args.prof, sizeof(unsigned long long) * 8 * grid);
    kern<<<grid, kK8Threads, smem, s>>>(dz_map, w_map, args);
    if (cudaGetLastError() != cudaSuccess) return cudaErrorUnknown;
    if (prof) {  // diagnostics: mean per-CTA cycle split (stderr)
        std::vector<unsigned long long> hh(8 * grid);
        cudaStreamSynchronize(s);
        cudaMemcpy(hh.data(), args.prof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost);
        double m[8] = {};
        for (int c = 0; c < grid; ++c)
            for (int k = 0; k < 8; ++k) m[k] += static_cast<double>(hh[c * 8 + k]) / grid;
        fprintf(stderr, "K8 grid %d stages %d | cycles/CTA %.0f | producer wait empty %.0f | MMA wait full %.0f, acc_empty %.0f"
                        " | epilogue wait acc_full %.0f, end %.0f | tiles/CTA %.0f\n", grid, stages, m[0], m[1], m[2], m[3], m[4], m[5], m[6]);
        cudaFree(args.prof);
    }
    return cudaGetLastError();
}

cudaError_t launch_k9(const __nv_bfloat16* dz, const __nv_bfloat16* h, int R, int H, int Hg, int V, int Vp,
                      float* part, float* d_weight, float* d_bias, cudaStream_t s, int max_ctas) {
    int smem_max = 0;
    const int nsm = sm_count_and_smem(&smem_max);
    if (!nsm) return cudaErrorUnknown;
    const int nvt = Vp / 128;
    const char* e9 = getenv("RNNT_K9_CLUSTER");  // A/B: a single-CTA cluster size (1, 2, 4, 8) instead of pairs
    const bool pair = !e9;
    int cl = pair ? 2 : std::max(1, std::min(std::min(cluster_for(H / 64, 8), 8), atoi(e9)));
    while (!pair && cl > 1 && cl > nvt) cl /= 2;
    const int groups = (nvt + cl - 1) / cl;
    const int64_t nst_total = (static_cast<int64_t>(std::max(R, 0)) + kK9Rows - 1) / kK9Rows;
    const int slot = (2 + (pair ? H / 128 : H / 64)) * kK9Box;
    int stages = kBwdMaxStages;
    auto smem_of = [&](int st) { return static_cast<size_t>(1024 + st * slot + (3 * kBwdMaxStages + 2) * 8 + 4096); };
    while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
    const size_t smem = smem_of(stages);
    auto kern = pair ? k9_dw_2sm<0> : cl == 8 ? k9_dw<8> : cl == 4 ? k9_dw<4> : cl == 2 ? k9_dw<2> : k9_dw<1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return cudaErrorInvalidConfiguration;
    int resident = max_clusters(kern, cl, smem, kK9Threads);  // one wave: every work unit co-resident
    if (resident <= 0) resident = nsm / cl;
    if (max_ctas > 0) resident = std::max(1, std::min(resident, max_ctas / cl));  // leave SMs to a concurrent K7
    int splits = std::max(1, std::min(resident, kK9MaxCtas / cl) / groups);
    splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(splits, nst_total)));
    const int per = static_cast<int>((nst_total + splits - 1) / splits);
    float* part_b = part + static_cast<size_t>(splits) * Vp * H;
    if (R > 0) {
        CUtensorMap dz_map, h_map;
        if (!make_map(&dz_map, dz, Vp, R, Vp, 64, kK9Rows) || !make_map(&h_map, h, H, R, Hg, 64, kK9Rows))
            return cudaErrorUnknown;
        K9Args args{part, part_b, R, H, Vp, nvt, groups, splits, per, stages, 0, nullptr};
        if (const char* e = getenv("RNNT_K9_DEBUG")) args.dbg = atoi(e);
        const int grid = splits * groups * cl;
        if (args.dbg & 4) cudaMalloc(&args.prof, sizeof(unsigned long long) * 8 * grid);
        kern<<<grid, kK9Threads, smem, s>>>(dz_map, h_map, args);
        if (cudaGetLastError() != cudaSuccess) return cudaErrorUnknown;
        if (args.prof) {  // diagnostics: mean per-CTA cycle split (stderr)
            unsigned long long h[8 * kK9MaxCtas] = {};
            cudaStreamSynchronize(s);
            cudaMemcpy(h, args.prof, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost);
            double m[8] = {};
            for (int c = 0; c < grid; ++c)
                for (int k = 0; k < 8; ++k) m[k] += static_cast<double>(h[c * 8 + k]) / grid;
            fprintf(stderr, "K9 grid %d stages %d | cycles/CTA producer %.0f (wait empty %.0f) | leader MMA wait full %.0f (x2) | "
                            "dbias wait mma_done %.0f | epilogue end %.0f | stages/CTA %.0f\n", grid, stages, m[0], m[1], 2 * m[2], m[3], m[4], m[5]);
            cudaFree(args.prof);
        }
    } else {
        splits = 1;
        if (cudaMemsetAsync(part, 0, sizeof(float) * (static_cast<size_t>(Vp) * H + Vp), s) != cudaSuccess)
            return cudaErrorUnknown;
        part_b = part + static_cast<size_t>(Vp) * H;
    }
    k9_reduce<<<nsm * 4, 256, 0, s>>>(part, part_b, splits, V, Vp, H, d_weight, d_bias);
    return cudaGetLastError();
}

}  // namespace rnnt
