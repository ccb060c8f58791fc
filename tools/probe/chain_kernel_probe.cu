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
    size_t smem = (size_t)S * 3 * T * P * 8 + 2 * S * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<(nch + 63) / 64, 96, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<(nch + 63) / 64, 96, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return ms / 10;
}

int main() {
    const int n = 16384, P = 8, p = 8;
    double *s0, *s1, *s2, *out;
    cudaMalloc(&s0, n * P * 8);
    cudaMalloc(&s1, n * P * 8);
    cudaMalloc(&s2, n * P * 8);
    cudaMalloc(&out, 4096 * 8);
    cudaMemset(s0, 0, n * P * 8);
    cudaMemset(s1, 0, n * P * 8);
    cudaMemset(s2, 0, n * P * 8);
    std::vector<ChainDesc> h;
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) h.push_back(ChainDesc{0, (uint8_t)i, 1, (uint8_t)j, (uint16_t)(i * P + j), 0, 0});
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) h.push_back(ChainDesc{2, (uint8_t)i, 0, (uint8_t)j, (uint16_t)(64 + i * P + j), 1, 0});
    for (int i = 0; i < p; ++i) h.push_back(ChainDesc{0, (uint8_t)i, 0, (uint8_t)i, (uint16_t)(128 + i), 0, 0});
    ChainDesc* d;
    cudaMalloc(&d, h.size() * sizeof(ChainDesc));
    cudaMemcpy(d, h.data(), h.size() * sizeof(ChainDesc), cudaMemcpyHostToDevice);
    const int nch = (int)h.size();
    for (int w = 0; w < 2; ++w) {
        std::printf("T=64  S=6 : %8.1f us\n", 1e3 * run<8, 64, 6>(s0, s1, s2, n, d, nch, out));
        std::printf("T=64  S=3 : %8.1f us\n", 1e3 * run<8, 64, 3>(s0, s1, s2, n, d, nch, out));
        std::printf("T=128 S=4 : %8.1f us\n", 1e3 * run<8, 128, 4>(s0, s1, s2, n, d, nch, out));
        std::printf("T=32  S=8 : %8.1f us\n", 1e3 * run<8, 32, 8>(s0, s1, s2, n, d, nch, out));
        std::printf("T=256 S=2 : %8.1f us\n", 1e3 * run<8, 256, 2>(s0, s1, s2, n, d, nch, out));
    }
    std::printf("(chain of %d steps: %.1f us at 12 cycles/step, 1.9 GHz)\n", n, n * 12 / 1.9e3);
    return 0;
}
