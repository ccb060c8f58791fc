// fp64_lat_probe.cu -- single-warp FP64 latency / issue microbenchmark
// (refgen chain design): cycles per dependent DADD, per independent DMUL,
// and per step of a mixed body (3 independent FP64 ops + 1 chain DADD).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, double x, int iters, long long* cyc) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) a = __dadd_rn(a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_indep(double* out, double x, int iters, long long* cyc) {
    double a[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) a[u] = x + u;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int u = 0; u < 16; ++u) a[u] = __dmul_rn(a[u], x);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) s += a[u];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// mixed: chain DADD + 3 independent FP64 ops per step on 16 independent lanes of work
__global__ void k_mixed(double* out, double x, int iters, long long* cyc) {
    double acc = 0, v[16], c = x * 0.25;
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = x + u;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            double y = __dsub_rn(v[u & 15], __dmul_rn(c, v[(u + 3) & 15]));
            v[u & 15] = y;
            acc = __dadd_rn(acc, __dmul_rn(y, c));
        }
    }
    long long t1 = clock64();
    double s = acc;
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    long long h;
    for (int w = 1; w <= 4; w *= 2) {
        k_chain<<<1, 32 * w>>>(out, 1.0001, iters, cyc);
        cudaDeviceSynchronize();
        k_chain<<<1, 32 * w>>>(out, 1.0001, iters, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps=%d dependent DADD: %.2f cycles each\n", w, (double)h / (iters * 32.0));
        k_indep<<<1, 32 * w>>>(out, 1.0001, iters, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps=%d independent DMUL (per warp): %.2f cycles each\n", w, (double)h / (iters * 32.0));
        k_mixed<<<1, 32 * w>>>(out, 1.0001, iters, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps=%d mixed step (DMUL,DSUB,DMUL indep + chain DADD): %.2f cycles/step\n", w,
               (double)h / (iters * 32.0));
    }
    return 0;
}
