// Sweep ad_exact_kernel configurations at the cfg-2 shape (n=16384, P=8) and
// others: time per launch (CUDA events, A = 2.15 GB > L2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o ad_probe ad_probe.cu
#include <cstdio>
#include "exact_kernels.cuh"

using namespace coopcg_gpu;

template <int P, int CPT, int BR, int T, int S, int RPT = 1>
void run(const double* Ap, int n, const double* D, double* Y, int p) {
    auto k = (RPT == 1) ? ad_exact_kernel<P, CPT, BR, T, S> : ad_exact_rpt_kernel<P, CPT, BR, T, S, 2>;
    size_t smem = (size_t)S * T * (BR + P) * 8 + 2 * S * 8;
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((n + BR - 1) / BR), block(32 + 32 * ad_consumer_warps(BR / RPT, P / CPT));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<grid, block, smem>>>(Ap, n, n, 0, D, Y, nullptr, p, nullptr, PeerRows{});
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k<<<grid, block, smem>>>(Ap, n, n, 0, D, Y, nullptr, p, nullptr, PeerRows{});
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    cudaError_t e = cudaGetLastError();
    std::printf("n=%6d P=%2d CPT=%d RPT=%d BR=%3d T=%3d S=%d smem=%6zu : %8.3f ms  %7.1f GB/s  %5.2f TF/s %s\n", n, P,
                CPT, RPT, BR, T, S, smem, ms, 8.0 * n * n / (ms * 1e-3) / 1e9, 2.0 * n * n * p / (ms * 1e-3) / 1e12,
                e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char** argv) {
    // argv[1]: "big" sweeps the P = 16 / 32 configurations at the cfg 3 / 4 sizes
    const bool big = argc > 1 && argv[1][0] == 'b';
    const int n = big ? 65536 : 16384;
    double *Ap, *D, *Y;
    const size_t nmax = big ? 131072 : 16384;
    cudaMalloc(&Ap, nmax * nmax * 8 + (size_t)128 * nmax * 8);
    cudaMalloc(&D, nmax * 32 * 8);
    cudaMalloc(&Y, nmax * 32 * 8);
    cudaMemset(Ap, 0, nmax * nmax * 8);
    cudaMemset(D, 0, nmax * 32 * 8);
    if (big) {
        run<16, 4, 64, 32, 4, 2>(Ap, n, D, Y, 16);
        run<16, 4, 64, 64, 2, 2>(Ap, n, D, Y, 16);
        run<16, 4, 64, 64, 3, 2>(Ap, n, D, Y, 16);
        run<16, 4, 64, 128, 2, 2>(Ap, n, D, Y, 16);
        run<16, 4, 128, 64, 2, 2>(Ap, n, D, Y, 16);
        const int n4 = 131072;
        run<32, 4, 64, 32, 4, 2>(Ap, n4, D, Y, 32);
        run<32, 4, 64, 64, 2, 2>(Ap, n4, D, Y, 32);
        run<32, 4, 64, 64, 3, 2>(Ap, n4, D, Y, 32);
        run<32, 4, 128, 64, 2, 2>(Ap, n4, D, Y, 32);
        return 0;
    }
    run<8, 4, 64, 32, 4, 1>(Ap, n, D, Y, 8);
    run<4, 2, 32, 32, 4, 1>(Ap, n, D, Y, 4);
    run<4, 2, 32, 32, 4, 1>(Ap, 4096, D, Y, 4);
    run<4, 2, 32, 64, 2, 1>(Ap, 4096, D, Y, 4);
    run<4, 2, 32, 32, 2, 1>(Ap, 4096, D, Y, 4);
    return 0;
}
