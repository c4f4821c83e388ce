// Microbenchmark: tcgen05.mma.cta_group::1.kind::f16 issue rate for operand majors (K / MN) of A and B in
// shared memory (SWIZZLE_128B descriptors), M = 128, N = 256, K = 16 per instruction, fp32 accumulate.
// Data are zeros (rate does not depend on values).  One CTA per SM; prints cycles per MMA (ideal: 128).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2303_10384_b200/csrc -I ../../include mma_rate.cu -o mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace rnnt;

__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

__global__ void __launch_bounds__(128, 1) bench(int amn, int bmn, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        const uint32_t sa = smem_u32(base), sb = smem_u32(base + 32768);
        const uint32_t id = idesc_bf16(128, 256, amn, bmn);
        // A: 128 x 16 per MMA; K-major: 128 rows of 128 B (SBO 1024), step 32 B; MN-major: 2 blocks of 64 (LBO 8 KB), step 2048 B
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < 16; ++k) {
                const uint64_t ad = amn ? sw128_mn_desc(sa + (k & 3) * 2048, 8192) : sw128_desc(sa) + 2 * (k & 3);
                const uint64_t bd = bmn ? sw128_mn_desc(sb + (k & 3) * 2048, 8192) : sw128_desc(sb) + 2 * (k & 3);
                mma1(tmem, ad, bd, id, k);
            }
            tc_commit(&bar);
            mbar_wait(&bar, ph);
            ph ^= 1;
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 2000;
    for (int amn = 0; amn < 2; ++amn)
        for (int bmn = 0; bmn < 2; ++bmn) {
            bench<<<148, 128, 100 * 1024>>>(amn, bmn, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < 148; ++i) m += h[i];
            m /= 148;
            printf("A %s B %s: %.1f cycles per 128x256x16 MMA (%s)\n", amn ? "MN" : "K ", bmn ? "MN" : "K ", m / (iters * 16.0),
                   cudaGetErrorString(e));
        }
    return 0;
}
