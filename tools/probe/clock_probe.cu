// Cycles per step of the production chain kernel vs wall time: run it with a
// side kernel that samples %clock64 and %globaltimer on the same SMs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o clock_probe clock_probe.cu
#include <cstdio>
#include <vector>
#include "exact_kernels.cuh"
using namespace coopcg_gpu;

__global__ void clk(unsigned long long* out, int spins) {
    unsigned long long c0 = clock64(), t0 = globaltimer_ns();
    double x = 1.0;
    for (int i = 0; i < spins; ++i) x = __dadd_rn(x, 1e-9);
    unsigned long long c1 = clock64(), t1 = globaltimer_ns();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = t1 - t0; if (x == 0) out[2] = 1; }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 32);
    for (int light = 0; light < 2; ++light) {
        clk<<<light ? 3 : 1, 32>>>(d, 2000000);
        unsigned long long h[3];
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        std::printf("%s: %.0f cycles in %.0f ns -> %.3f GHz; %.2f cycles per dependent DADD\n",
                    light ? "3 CTAs" : "1 CTA", (double)h[0], (double)h[1], (double)h[0] / h[1],
                    (double)h[0] / 2000000);
    }
    return 0;
}
