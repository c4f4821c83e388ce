// Microbenchmark: producer / consumer cadence of an mbarrier ring without data: warp 0 waits empty[s] and
// arrives on full[s]; warp 1 waits full[s] and releases empty[s] either by tcgen05.commit (mode 0) or by a plain
// arrive (mode 1); optionally (mode 2) warps 4-7 also wait on a commit-signalled barrier and arrive on empty.
// Prints cycles per stage for stages = 2, 4, 8.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I /root/repo/paper_2303_10384_b200/csrc -I /root/repo/include pipe_rate.cu -o pipe_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace rnnt;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) bench2(int mode, int stages, int iters, unsigned long long* out) {
    // the K9 pair ring: both producers wait their empty[s]; the leader's arrives on its full[s]; the leader's
    // MMA warp waits full[s] and commits (cta_group::2, multicast to both CTAs) to done[s]; each CTA's 4 warps
    // wait done[s] and arrive on their empty[s].  mode 1: the commit is replaced by two remote arrives.
    __shared__ uint64_t full[8], empty[8], done[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = static_cast<int>(cluster_rank());
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
            mbar_init(&done[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc_2sm(&slot, 32);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            if (rank == 0) mbar_arrive(&full[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1 && rank == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (mode == 0) tc_commit_2sm_mc(&done[s], 3);
            else if (lane == 0) { mbar_arrive(&done[s]); mbar_arrive_remote(&done[s], 1); }
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (warp >= 4) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&done[s], ph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_2sm(slot, 32);
}

__global__ void __launch_bounds__(256, 1) bench(int mode, int stages, int iters, unsigned long long* out) {
    __shared__ uint64_t full[8], empty[8], done[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], mode == 2 ? 4 : 1);
            mbar_init(&done[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive(&full[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (mode == 0) tc_commit(&empty[s]);
            else if (mode == 1) { if (lane == 0) mbar_arrive(&empty[s]); }
            else tc_commit(&done[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (warp >= 4 && mode == 2) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&done[s], ph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(32) : "memory");
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int iters = 20000;
    const char* names[3] = {"commit->empty", "arrive->empty", "commit->done->4 warps->empty"};
    for (int mode = 0; mode < 3; ++mode)
        for (int st = 2; st <= 8; st *= 2) {
            bench<<<148, 256>>>(mode, st, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < 148; ++i) m += h[i];
            printf("%-32s stages %d: %.1f cycles per stage (%s)\n", names[mode], st, m / 148 / iters, cudaGetErrorString(e));
        }
    const char* n2[2] = {"pair: commit.cta_group::2 mc", "pair: two plain arrives"};
    for (int mode = 0; mode < 2; ++mode)
        for (int st = 2; st <= 8; st *= 2) {
            bench2<<<148, 256>>>(mode, st, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < 148; ++i) m += h[i];
            printf("%-32s stages %d: %.1f cycles per stage (%s)\n", n2[mode], st, m / 148 / iters, cudaGetErrorString(e));
        }
    return 0;
}
