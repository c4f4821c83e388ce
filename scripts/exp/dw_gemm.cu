// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o scripts/exp/dw_gemm scripts/exp/dw_gemm.cu -lcublas
// Shape experiment for the joint backward's dW GEMM: [M x V] = A[M x R] . B[R x V]^T-view, bf16 in, fp32 out.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
    const long R = argc > 1 ? atol(argv[1]) : 1616000;
    const int V = argc > 2 ? atoi(argv[2]) : 1024;
    cublasHandle_t h;
    cublasCreate(&h);
    const int Ms[] = {512, 520, 528, 576, 640};
    for (int M : Ms) {
        void *a, *b, *c;
        cudaMalloc(&a, (size_t)R * M * 2);
        cudaMalloc(&b, (size_t)R * V * 2);
        cudaMalloc(&c, (size_t)M * V * 4);
        cudaMemset(a, 0, (size_t)R * M * 2);
        cudaMemset(b, 0, (size_t)R * V * 2);
        float one = 1.f, zero = 0.f;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int it = 0; it < 3; ++it)
            cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, M, V, R, &one, a, CUDA_R_16BF, M, b, CUDA_R_16BF, V, &zero, c,
                         CUDA_R_32F, M, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it)
            cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_T, M, V, R, &one, a, CUDA_R_16BF, M, b, CUDA_R_16BF, V, &zero, c,
                         CUDA_R_32F, M, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        printf("M=%d V=%d R=%ld: %.3f ms  %.0f TF/s (on M)  %.0f TF/s (on 512)\n", M, V, R, ms,
               2.0 * M * V * R / ms / 1e9, 2.0 * 512 * V * R / ms / 1e9);
        // dh-type GEMM for reference: [512 x R] = W^T[512 x V] . dz^T [V x R]
        cudaFree(a);
        cudaFree(b);
        cudaFree(c);
    }
    return 0;
}
