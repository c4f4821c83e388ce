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
// Operands (bf16, fp32 accumulation in TMEM): dz [R][Vp] and h [R][Hg] as K6<grad> writes them, W [V][H] as the
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

// =============================================================================================== K8 (dh)
constexpr int kK8Threads = 384;  // warps: 0 TMA, 1 MMA, 2-3 idle, 4-11 epilogue (2 per TMEM lane quarter)
constexpr int kK8KBlock = 64;    // v per stage (one 128-byte swizzle row of the K-major A)
constexpr int kK8ABytes = 128 * kK8KBlock * 2;      // dz box {64 v, 128 rows}
constexpr int kK8BBox = kK8KBlock * 64 * 2;          // W box {64 h, 64 v}

struct K8Args {
    const __nv_bfloat16* h;   // [R][Hg]
    __nv_bfloat16* dpre;      // [R][H]
    int R, H, Hg, V, stages;
};

template <int kCl>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kK8Threads, 1)
    k8_dh_tanh(const __grid_constant__ CUtensorMap dz_map, const __grid_constant__ CUtensorMap w_map, const K8Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int H = a.H, nbox = H / 64;
    const int slot_bytes = kK8ABytes + nbox * kK8BBox;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(a.stages) * slot_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kBwdMaxStages;
    uint64_t* acc_full = bars + 2 * kBwdMaxStages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCl);  // released by the MMAs of every CTA of the cluster
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 256);
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
    const int64_t bx = blockIdx.x, cl0 = bx - bx % kCl;
    const int64_t n_iter = ntiles > cl0 ? (ntiles - cl0 + gridDim.x - 1) / gridDim.x : 0;  // the cluster's count
    const uint32_t crank = kCl > 1 ? cluster_rank() : 0;
    const int KB = (a.V + kK8KBlock - 1) / kK8KBlock;  // dz's columns past V are zero: K stops at V

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: own dz box + 1/kCl of the W boxes, multicast =====
            int s = 0;
            uint32_t ph = 0;
            for (int64_t k = 0; k < n_iter; ++k) {
                const int64_t r0 = (bx + k * gridDim.x) * 128;
                const bool a_in = r0 < a.R;  // a dummy tile past the end (the cluster's lockstep): no A load
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], slot_bytes - (a_in ? 0 : kK8ABytes));
                    uint8_t* slot = base + static_cast<size_t>(s) * slot_bytes;
                    if (a_in) tma_load_2d(slot, &dz_map, &full[s], kb * kK8KBlock, static_cast<int>(r0));
                    for (int j = static_cast<int>(crank); j < nbox; j += kCl) {
                        uint8_t* dst = slot + kK8ABytes + j * kK8BBox;
                        if constexpr (kCl > 1)
                            tma_load_2d_mc(dst, &w_map, &full[s], j * 64, kb * kK8KBlock,
                                           static_cast<uint16_t>((1u << kCl) - 1));
                        else
                            tma_load_2d(dst, &w_map, &full[s], j * 64, kb * kK8KBlock);
                    }
                    if (++s == a.stages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: D[128 rows x H] (+)= dz[128 x 64] . W[64 x H] per stage, N in chunks of <= 256 =====
        int s = 0;
        uint32_t ph = 0;
        for (int64_t k = 0; k < n_iter; ++k) {
            mbar_wait(acc_empty, (static_cast<uint32_t>(k) & 1) ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t sa = smem_u32(base + static_cast<size_t>(s) * slot_bytes);
                const uint64_t adesc = sw128_desc(sa);
#pragma unroll
                for (int ks = 0; ks < kK8KBlock / 16; ++ks)
                    for (int n0 = 0; n0 < H; n0 += 256) {
                        const int N = min(256, H - n0);
                        const uint64_t bdesc = sw128_mn_desc(sa + kK8ABytes + (n0 / 64) * kK8BBox + ks * 2048, kK8BBox);
                        mma_ss(tmem + n0, adesc + 2 * ks, bdesc, idesc_bf16(128, N, false, true), (kb | ks) ? 1u : 0u);
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
        }
    } else if (warp >= 4) {
        // ===== epilogue: thread = row (TMEM lane); the two warps of a lane quarter split the H columns =====
        const int q = warp & 3, eh = (warp - 4) >> 2;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
        const int c_lo = eh * (H / 2), c_hi = c_lo + H / 2;
        for (int64_t k = 0; k < n_iter; ++k) {
            const int64_t row = (bx + k * gridDim.x) * 128 + q * 32 + lane;
            const bool live = row < a.R;
            mbar_wait(acc_full, static_cast<uint32_t>(k) & 1);
            tc_fence_after();
            const __nv_bfloat16* hr = a.h + row * a.Hg;
            __nv_bfloat16* out = a.dpre + row * H;
            for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
                uint32_t r[32];
                uint4 hv[4];
                if (live) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) hv[i] = __ldcs(reinterpret_cast<const uint4*>(hr + c0) + i);
                }
                TMEM_LD32(lane_base + c0, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (live) {
                    uint4 o[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t hw[4] = {hv[i].x, hv[i].y, hv[i].z, hv[i].w};
                        uint32_t ow[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 hh = unpack_bf16x2(hw[j]);
                            const float2 d = upk(fmul2(pk(__uint_as_float(r[8 * i + 2 * j]), __uint_as_float(r[8 * i + 2 * j + 1])),
                                                      ffma2(pk(-hh.x, -hh.y), pk(hh.x, hh.y), pk(1.f, 1.f))));
                            ow[j] = pack_bf16x2(d.x, d.y);
                        }
                        o[i] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) __stcs(reinterpret_cast<uint4*>(out + c0) + i, o[i]);
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty);
        }
    }
    tc_fence_before();
    if constexpr (kCl > 1)
        cluster_sync_all();  // no CTA leaves while a partner may still multicast into it
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, kBwdTmemCols);
}

// =============================================================================================== K9 (dW)
constexpr int kK9Threads = 384;  // warps: 0 TMA, 1 MMA, 2-3 idle, 4-7 dbias summers, 8-11 epilogue
constexpr int kK9Rows = 32;      // K (rows) per stage
constexpr int kK9Box = 64 * kK9Rows * 2;  // one {64 elements, 32 rows} box, 4 KB
constexpr int kK9MaxCtas = 256;

struct K9Args {
    float* part;    // [splits][Vp][H] fp32 partial dW
    float* part_b;  // [splits][Vp] partial dbias
    int R, H, Vp, nvt, groups, splits, stages_per_split, stages;
};

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
        const int vl = threadIdx.x - 128, box = vl >> 6, c = vl & 63;
        float acc = 0.f;
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nst; ++i) {
            mbar_wait(&full[s], ph);
            const uint8_t* bb = base + static_cast<size_t>(s) * slot_bytes + box * kK9Box + ((c & 7) << 1);
#pragma unroll 8
            for (int k = 0; k < kK9Rows; ++k) {
                const uint16_t v = *reinterpret_cast<const uint16_t*>(bb + k * 128 + ((((c >> 3) ^ (k & 7))) << 4));
                acc += __uint_as_float(static_cast<uint32_t>(v) << 16);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        if (vt < a.nvt) a.part_b[static_cast<int64_t>(split) * a.Vp + v0 + vl] = acc;
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
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s = 0; s < splits; ++s) {
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
                      __nv_bfloat16* dpre, int R, int H, int Hg, int V, int Vp, cudaStream_t s) {
    if (R <= 0) return cudaSuccess;
    int smem_max = 0;
    const int nsm = sm_count_and_smem(&smem_max);
    if (!nsm) return cudaErrorUnknown;
    CUtensorMap dz_map, w_map;
    if (!make_map(&dz_map, dz, Vp, R, Vp, kK8KBlock, 128) || !make_map(&w_map, weight, H, V, H, 64, kK8KBlock))
        return cudaErrorUnknown;
    const int nbox = H / 64, slot = kK8ABytes + nbox * kK8BBox;
    int stages = kBwdMaxStages;
    auto smem_of = [&](int st) { return static_cast<size_t>(1024 + st * slot + (2 * kBwdMaxStages + 2) * 8 + 16); };
    while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
    const size_t smem = smem_of(stages);
    if (smem > static_cast<size_t>(smem_max)) return cudaErrorInvalidConfiguration;
    int cl = cluster_for(nbox, 4);
    if (const char* e = getenv("RNNT_K8_CLUSTER")) cl = std::max(1, std::min(cl, atoi(e)));
    auto kern = cl == 4 ? k8_dh_tanh<4> : cl == 2 ? k8_dh_tanh<2> : k8_dh_tanh<1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return cudaErrorInvalidConfiguration;
    const int64_t ntiles = (static_cast<int64_t>(R) + 127) / 128;
    int resident = max_clusters(kern, cl, smem, kK8Threads) * cl;  // persistent: only co-resident clusters
    if (resident <= 0) resident = nsm - nsm % cl;
    int grid = static_cast<int>(std::min<int64_t>(ntiles, resident));
    grid = std::max(cl, grid - grid % cl);
    K8Args args{h, dpre, R, H, Hg, V, stages};
    kern<<<grid, kK8Threads, smem, s>>>(dz_map, w_map, args);
    return cudaGetLastError();
}

cudaError_t launch_k9(const __nv_bfloat16* dz, const __nv_bfloat16* h, int R, int H, int Hg, int V, int Vp,
                      float* part, float* d_weight, float* d_bias, cudaStream_t s) {
    int smem_max = 0;
    const int nsm = sm_count_and_smem(&smem_max);
    if (!nsm) return cudaErrorUnknown;
    const int nvt = Vp / 128;
    int cl = std::min(cluster_for(H / 64, 8), 8);
    while (cl > 1 && cl > nvt) cl /= 2;
    if (const char* e = getenv("RNNT_K9_CLUSTER")) cl = std::max(1, std::min(cl, atoi(e)));
    const int groups = (nvt + cl - 1) / cl;
    const int64_t nst_total = (static_cast<int64_t>(std::max(R, 0)) + kK9Rows - 1) / kK9Rows;
    const int slot = (2 + H / 64) * kK9Box;
    int stages = kBwdMaxStages;
    auto smem_of = [&](int st) { return static_cast<size_t>(1024 + st * slot + (2 * kBwdMaxStages + 1) * 8 + 16); };
    while (stages > 2 && smem_of(stages) > static_cast<size_t>(smem_max)) --stages;
    const size_t smem = smem_of(stages);
    auto kern = cl == 8 ? k9_dw<8> : cl == 4 ? k9_dw<4> : cl == 2 ? k9_dw<2> : k9_dw<1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return cudaErrorInvalidConfiguration;
    int resident = max_clusters(kern, cl, smem, kK9Threads);  // one wave: every work unit co-resident
    if (resident <= 0) resident = nsm / cl;
    int splits = std::max(1, std::min(resident, kK9MaxCtas / cl) / groups);
    splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(splits, nst_total)));
    const int per = static_cast<int>((nst_total + splits - 1) / splits);
    float* part_b = part + static_cast<size_t>(splits) * Vp * H;
    if (R > 0) {
        CUtensorMap dz_map, h_map;
        if (!make_map(&dz_map, dz, Vp, R, Vp, 64, kK9Rows) || !make_map(&h_map, h, H, R, Hg, 64, kK9Rows))
            return cudaErrorUnknown;
        K9Args args{part, part_b, R, H, Vp, nvt, groups, splits, per, stages};
        kern<<<splits * groups * cl, kK9Threads, smem, s>>>(dz_map, h_map, args);
        if (cudaGetLastError() != cudaSuccess) return cudaErrorUnknown;
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
