// A/B timing of the exact A.D kernel: current header vs the pre-RPT header
// (old_exact_ad.cuh, generated from git 3d29d19) on the same box.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o ad_cmp_probe ad_cmp_probe.cu
#include <cstdio>
#include "exact_kernels.cuh"
#include "old_exact_ad.cuh"

template <typename K>
float timeit(K k, dim3 grid, dim3 block, size_t smem, const double* Ap, int n, const double* D, double* Y, int p) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<grid, block, smem>>>(Ap, n, n, 0, D, Y, nullptr, p, nullptr);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<grid, block, smem>>>(Ap, n, n, 0, D, Y, nullptr, p, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10;
}

int main() {
    const int n = 16384;
    double *Ap, *D, *Y;
    cudaMalloc(&Ap, (size_t)n * n * 8 + (size_t)128 * n * 8);
    cudaMalloc(&D, (size_t)n * 32 * 8);
    cudaMalloc(&Y, (size_t)n * 32 * 8);
    cudaMemset(Ap, 0, (size_t)n * n * 8);
    cudaMemset(D, 0, (size_t)n * 32 * 8);
    const size_t smem = (size_t)4 * 32 * (64 + 8) * 8 + 2 * 4 * 8;
    dim3 grid(n / 64), block(32 + 64 * 2);
    for (int w = 0; w < 3; ++w) {
        float tn = timeit(coopcg_gpu::ad_exact_kernel<8, 4, 64, 32, 4>, grid, block, smem, Ap, n, D, Y, 8);
        float to = timeit(coopcg_old::ad_exact_kernel<8, 4, 64, 32, 4>, grid, block, smem, Ap, n, D, Y, 8);
        std::printf("new %.1f us   old %.1f us  %s\n", tn * 1e3, to * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
