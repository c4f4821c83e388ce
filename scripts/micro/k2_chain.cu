// Microbenchmark: the dependent chain of one K2 wavefront step (one warp, kC cells per lane, neighbour by
// shuffle), in registers only, for variants of the log-sum-exp.  Prints ns per step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I /root/repo/paper_2303_10384_b200/csrc -I /root/repo/include k2_chain.cu -o k2_chain
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace rnnt;

// variant 1: lse in fp64 with a fp32 correction computed from the fp64 difference (current K2)
__device__ __forceinline__ double lse_v1(double a, double b) { return lse2f(a, b); }
// variant 2: the max / difference in fp64 but the correction from fp32 copies of a and b kept alongside
// (no F2F on the chain: af, bf are separate fp32 registers updated with the value) -- modelled as converting
// once per step outside the chain
__device__ __forceinline__ double lse_v2(double a, double b, float af, float bf) {
    const double m = a > b ? a : b;
    const float x = -fabsf(af - bf) * kLog2e;
    const float c = lg2(1.f + ex2(x)) * kLn2;
    return m + static_cast<double>(c);
}
// variant 3: everything in fp32 (the precision R11 rejects; lower bound of the chain)
__device__ __forceinline__ float lse_v3(float a, float b) {
    const float m = fmaxf(a, b);
    const float c = lg2(1.f + ex2(-fabsf(a - b) * kLog2e)) * kLn2;
    return m + c;
}

// variant 4: fp64 values and adds, everything else on the integer / fp32 pipes: the max from the sign bit of
// the fp64 difference, the fp32 copy of -|diff| and the fp64 copy of the fp32 correction by bit manipulation
// (no DSETP, no F2F: the FP64 pipe only sees the adds).
__device__ __forceinline__ float f32_of_negabs_f64(double d) {
    // -|d| as fp32 (truncating the mantissa; exact enough: the correction's slope is <= 0.5), clamped to
    // [-64, 0]: |d| >= 64 gives -64 (correction 2^-92: zero); tiny |d| (< 2^-126) gives -0.
    const unsigned long long bits = __double_as_longlong(d) & 0x7fffffffffffffffULL;
    const unsigned hi = static_cast<unsigned>(bits >> 32);
    if (hi >= 0x40500000u) return -64.f;                 // |d| >= 64 (also inf / NaN)
    if (hi < 0x38100000u) return -0.f;                   // |d| < 2^-126
    const unsigned e = (hi >> 20) - 1023u + 127u;
    const unsigned m = static_cast<unsigned>(bits >> 29) & 0x7fffffu;
    return __uint_as_float(0x80000000u | (e << 23) | m);
}
__device__ __forceinline__ double f64_of_f32_pos(float c) {   // c in [0, 1): exact widening by bits
    const unsigned b = __float_as_uint(c);
    if (b == 0u) return 0.0;
    const unsigned long long e = ((b >> 23) & 0xffu) - 127u + 1023u;
    return __longlong_as_double(static_cast<long long>((e << 52) | (static_cast<unsigned long long>(b & 0x7fffffu) << 29)));
}
__device__ __forceinline__ double lse_v4(double a, double b) {
    const double diff = a - b;
    const bool a_ge = static_cast<int>(__double2hiint(diff)) >= 0;   // sign bit of the difference (NaN: a)
    const double m = a_ge ? a : b;
    const float x = f32_of_negabs_f64(diff) * kLog2e;
    const float c = lg2(1.f + ex2(x)) * kLn2;
    return m + f64_of_f32_pos(c);
}

template <int V, int kC>
__global__ void chain(int steps, const double* x, double* out, long long* cyc) {
    double self[kC], pub[kC];
    float selff[kC], pubf[kC];
    for (int j = 0; j < kC; ++j) self[j] = pub[j] = -1.0 * (threadIdx.x + j), selff[j] = pubf[j] = (float)self[j];
    const double xb = x[threadIdx.x], xy = x[threadIdx.x + 32];
    long long t0 = clock64();
    for (int d = 0; d < steps; ++d) {
        double left = __shfl_up_sync(0xffffffffu, pub[kC - 1], 1);
        float leftf = __shfl_up_sync(0xffffffffu, pubf[kC - 1], 1);
#pragma unroll
        for (int j = kC - 1; j >= 0; --j) {
            const double nb = j == 0 ? left : pub[j - 1];
            if (V == 1) {
                const double cur = lse_v1(self[j], nb);
                self[j] = cur + xb;
                pub[j] = cur + xy;
            } else if (V == 2) {
                const float nbf = j == 0 ? leftf : pubf[j - 1];
                const double cur = lse_v2(self[j], nb, selff[j], nbf);
                self[j] = cur + xb;
                pub[j] = cur + xy;
                selff[j] = static_cast<float>(self[j]);
                pubf[j] = static_cast<float>(pub[j]);
            } else if (V == 5 || V == 7 || V == 8) {
                // restructured: the operand adds off the chain, (m + x) + c; V 7 / 8 add the kernel's per-cell
                // validity select (7: new form, 8: the current form cur + x)
                const int t = d - static_cast<int>(threadIdx.x) * kC - j;
                const bool valid = static_cast<unsigned>(t) < static_cast<unsigned>(steps);
                const double diff = self[j] - nb;
                const double m = diff > 0.0 ? self[j] : nb;
                const float xf = fminf(-fabsf(static_cast<float>(diff)) * kLog2e, 0.f);
                const double c = static_cast<double>(lg2(1.f + ex2(xf)) * kLn2);
                if (V == 5) {
                    self[j] = (m + xb) + c;
                    pub[j] = (m + xy) + c;
                } else if (V == 7) {
                    self[j] = valid ? (m + xb) + c : -INFINITY;
                    pub[j] = valid ? (m + xy) + c : -INFINITY;
                } else {
                    const double cur = m + c;
                    self[j] = valid ? cur + xb : -INFINITY;
                    pub[j] = valid ? cur + xy : -INFINITY;
                }
            } else if (V == 6) {
                // the current backward step: the neighbour's operand add and the terminal-cell select on the chain
                const int t = d - static_cast<int>(threadIdx.x) * kC - j;
                const bool valid = static_cast<unsigned>(t) < static_cast<unsigned>(steps);
                const bool last = t == steps - 3;
                const double op2 = nb + xy;
                double cur = lse_v1(self[j] + xb, op2);
                cur = last ? xb : cur;
                self[j] = valid ? cur : -INFINITY;
                pub[j] = self[j];
            } else if (V == 4) {
                const double cur = lse_v4(self[j], nb);
                self[j] = cur + xb;
                pub[j] = cur + xy;
            } else {
                const float nbf = j == 0 ? leftf : pubf[j - 1];
                const float cur = lse_v3(selff[j], nbf);
                selff[j] = cur + (float)xb;
                pubf[j] = cur + (float)xy;
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int j = 0; j < kC; ++j) s += self[j] + pub[j] + selff[j] + pubf[j];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *x, *o;
    long long* c;
    cudaMalloc(&x, 64 * 8); cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
    cudaMemset(x, 0, 64 * 8);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int steps = 100000;
    auto run = [&](auto kern, const char* name) {
        kern<<<1, 32>>>(steps, x, o, c);
        cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-44s %.1f cycles/step (%.1f ns at %d MHz)\n", name, (double)h / steps, (double)h / steps / (clk_khz / 1e6), clk_khz / 1000);
    };
    run(chain<1, 1>, "fp64 lse2f (K2 now), kC=1");
    run(chain<1, 2>, "fp64 lse2f (K2 now), kC=2");
    run(chain<2, 1>, "fp64 value, fp32 shadow for the correction, kC=1");
    run(chain<2, 2>, "fp64 value, fp32 shadow for the correction, kC=2");
    run(chain<3, 1>, "all fp32 (rejected by R11), kC=1");
    run(chain<4, 1>, "fp64 adds only (int max / conversions), kC=1");
    run(chain<4, 2>, "fp64 adds only (int max / conversions), kC=2");
    run(chain<5, 1>, "restructured (m + x) + c, kC=1");
    run(chain<5, 2>, "restructured (m + x) + c, kC=2");
    run(chain<8, 1>, "current forward + validity select, kC=1");
    run(chain<7, 1>, "restructured + validity select, kC=1");
    run(chain<6, 1>, "current backward (+x on chain, last select), kC=1");
    run(chain<8, 2>, "current forward + validity select, kC=2");
    run(chain<7, 2>, "restructured + validity select, kC=2");
    run(chain<6, 2>, "current backward (+x on chain, last select), kC=2");
    return 0;
}
