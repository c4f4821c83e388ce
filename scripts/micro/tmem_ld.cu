// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM with W warps (W/4 per TMEM lane quarter), loads only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I /root/repo/paper_2303_10384_b200/csrc -I /root/repo/include tmem_ld.cu -o tmem_ld
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace rnnt;

__global__ void __launch_bounds__(512, 1) bench(int iters, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int q = warp & 3, g = warp >> 2, nw = blockDim.x >> 5;
    const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
        TMEM_LD32(base + ((g * 32 + it * 32 * (nw / 4)) & 511), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 148 * 512 * 4);
    const int iters = 20000;
    for (int w = 4; w <= 16; w *= 2) {
        bench<<<148, w * 32>>>(iters, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < 148; ++i) m += h[i];
        m /= 148;
        const double bytes = double(iters) * w * 32 * 32 * 4;  // per SM
        printf("%2d warps: %.1f bytes/cycle/SM of tcgen05.ld (%s)\n", w, bytes / m, cudaGetErrorString(e));
    }
    return 0;
}
