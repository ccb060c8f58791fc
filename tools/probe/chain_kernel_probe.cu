// Time the production chain_kernel in isolation (P=8, three sources, the
// gram-phase chain set) for several (T, S) pipelines.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o chain_kernel_probe chain_kernel_probe.cu
#include <cstdio>
#include <vector>
#include "exact_kernels.cuh"

using namespace coopcg_gpu;

template <int P, int T, int S>
float run(const double* s0, const double* s1, const double* s2, int n, const ChainDesc* d, int nch, double* out) {
    auto k = chain_kernel<P, T, S>;
    size_t smem = chain_smem_bytes(P, T, S, 3);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<(nch + 63) / 64, kChainThreads, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<(nch + 63) / 64, kChainThreads, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return ms / 10;
}

template <int P>
void sweep(int n) {
    const int p = P;
    double *s0, *s1, *s2, *out;
    cudaMalloc(&s0, (size_t)n * P * 8);
    cudaMalloc(&s1, (size_t)n * P * 8);
    cudaMalloc(&s2, (size_t)n * P * 8);
    cudaMalloc(&out, 8192 * 8);
    cudaMemset(s0, 0, (size_t)n * P * 8);
    cudaMemset(s1, 0, (size_t)n * P * 8);
    cudaMemset(s2, 0, (size_t)n * P * 8);
    std::vector<ChainDesc> h;
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) h.push_back(ChainDesc{0, (uint8_t)i, 1, (uint8_t)j, (uint16_t)(i * P + j), 0, 0});
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) h.push_back(ChainDesc{2, (uint8_t)i, 0, (uint8_t)j, (uint16_t)(P * P + i * P + j), 1, 0});
    for (int i = 0; i < p; ++i) h.push_back(ChainDesc{0, (uint8_t)i, 0, (uint8_t)i, (uint16_t)(2 * P * P + i), 0, 0});
    ChainDesc* d;
    cudaMalloc(&d, h.size() * sizeof(ChainDesc));
    cudaMemcpy(d, h.data(), h.size() * sizeof(ChainDesc), cudaMemcpyHostToDevice);
    const int nch = (int)h.size();
#define R(T, S)                                                                                             \
    if (chain_smem_bytes(P, T, S, 3) <= 227 * 1024)                                                       \
        std::printf("P=%2d n=%d T=%3d S=%2d smem=%6zu : %8.1f us\n", P, n, T, S, chain_smem_bytes(P, T, S, 3), \
                    1e3 * run<P, T, S>(s0, s1, s2, n, d, nch, out));
    R(512, 3) R(384, 3) R(256, 4) R(256, 3) R(192, 3)
#undef R
    cudaFree(s0); cudaFree(s1); cudaFree(s2); cudaFree(out); cudaFree(d);
}

int main() {
    for (int w = 0; w < 2; ++w) {
        sweep<8>(16384);
        if (w == 1) { sweep<4>(16384); sweep<16>(16384); sweep<32>(16384); }
    }
    std::printf("(chain of 16384 steps: %.1f us at 9.4 cycles/step, 1.965 GHz)\n", 16384 * 9.4 / 1.965e3);
    return 0;
}
