// Dependent-chain latency microbenchmark (cycles per op) for ops on K2's critical path.
#include <cstdio>
#include <cstdint>
#define N 256
__global__ void k(double* outd, float* outf, long long* cyc, double seed) {
    double d = seed; float f = (float)seed; long long t0, t1; int iv = (int)seed;
    // DADD chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { d = d + 1e-9; d = d + 1e-9; d = d + 1e-9; d = d + 1e-9; }
    t1 = clock64(); cyc[0] = (t1 - t0); outd[0] = d;
    // F2F f64->f32->f64 roundtrip chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { f = (float)d; d = (double)f + 1e-9; f = (float)d; d = (double)f; }
    t1 = clock64(); cyc[1] = (t1 - t0); outd[1] = d;
    // MUFU.EX2 chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { asm volatile("ex2.approx.ftz.f32 %0,%0;" : "+f"(f)); asm volatile("ex2.approx.ftz.f32 %0,%0;" : "+f"(f)); asm volatile("ex2.approx.ftz.f32 %0,%0;" : "+f"(f)); asm volatile("ex2.approx.ftz.f32 %0,%0;" : "+f"(f)); }
    t1 = clock64(); cyc[2] = (t1 - t0); outf[0] = f;
    // FFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { f = fmaf(f, 1.0001f, 0.5f); f = fmaf(f, 1.0001f, 0.5f); f = fmaf(f, 1.0001f, 0.5f); f = fmaf(f, 1.0001f, 0.5f); }
    t1 = clock64(); cyc[3] = (t1 - t0); outf[1] = f;
    // SHFL chain (double)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); d = __shfl_up_sync(~0u, d, 1); }
    t1 = clock64(); cyc[4] = (t1 - t0); outd[2] = d;
    // DSETP+FSEL select chain (fmax)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { d = fmax(d, seed); d = fmax(d, seed+1); d = fmax(d, seed); d = fmax(d, seed+2); }
    t1 = clock64(); cyc[5] = (t1 - t0); outd[3] = d;
    // int add chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { iv = iv * 3 + 1; iv = iv * 3 + 1; iv = iv * 3 + 1; iv = iv * 3 + 1; }
    t1 = clock64(); cyc[6] = (t1 - t0); outd[4] = iv;
}
__global__ void kbar(long long* cyc, int nsteps) {
    __shared__ double s[32];
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < nsteps; ++i) {
        if ((threadIdx.x & 31) == 31) s[threadIdx.x >> 5] = v;
        asm volatile("bar.sync 1, %0;" :: "r"((int)blockDim.x) : "memory");
        if ((threadIdx.x & 31) == 0 && threadIdx.x) v += s[(threadIdx.x >> 5) - 1];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* od; float* of; long long* c; cudaMalloc(&od, 64); cudaMalloc(&of, 64); cudaMalloc(&c, 256);
    k<<<1, 32>>>(od, of, c, 1.5); long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* names[] = {"DADD", "F2F roundtrip (2 F2F per op... 4 conv per iter)", "MUFU.EX2", "FFMA", "SHFL.64", "DMNMX(fmax)", "IMAD"};
    for (int i = 0; i < 7; ++i) printf("%-50s %.1f cyc/op\n", names[i], h[i] / (4.0 * N));
    for (int nt : {32, 64, 128, 256}) {
        kbar<<<1, nt>>>(c, 1000); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("bar.sync step (STS+BAR+LDS) nthreads=%d: %.1f cyc/step\n", nt, h[0] / 1000.0);
    }
    return 0;
}
