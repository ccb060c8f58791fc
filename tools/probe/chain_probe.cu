// Microbenchmark: cycles per step of a sequential exact dot-product chain
// (acc = acc + x[k]*y[k], one rounding each) fed from shared memory, for
// several loop structures.  One CTA of 64 threads, each thread one chain over
// a 64-row x P tile re-walked `reps` times.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_probe chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int P = 8, T = 64;

__global__ void v0_naive(double* out, long long* cyc, int reps) {
    __shared__ double tile[2][T * P];
    for (int i = threadIdx.x; i < T * P; i += blockDim.x) { tile[0][i] = 1.0 + i * 1e-3; tile[1][i] = 0.5 - i * 1e-4; }
    __syncthreads();
    const double* xs = tile[0] + (threadIdx.x & 7);
    const double* ys = tile[1] + (threadIdx.x >> 3);
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 16
        for (int k = 0; k < T; ++k) acc = __dadd_rn(acc, __dmul_rn(xs[k * P], ys[k * P]));
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// batches of U with an un-unrolled batch loop: loads for batch b+1 at the top
template <int U>
__global__ void v1_batched(double* out, long long* cyc, int reps) {
    __shared__ double tile[2][T * P];
    for (int i = threadIdx.x; i < T * P; i += blockDim.x) { tile[0][i] = 1.0 + i * 1e-3; tile[1][i] = 0.5 - i * 1e-4; }
    __syncthreads();
    const double* xs = tile[0] + (threadIdx.x & 7);
    const double* ys = tile[1] + (threadIdx.x >> 3);
    double acc = 0.0;
    long long t0 = clock64();
    const int nb = reps * (T / U);
    double xv[U], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { xv[u] = xs[u * P]; yv[u] = ys[u * P]; }
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
        const int kn = ((b + 1) % (T / U)) * U;
        double nx[U], ny[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { nx[u] = xs[(kn + u) * P]; ny[u] = ys[(kn + u) * P]; }
        double pr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(xv[u], yv[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, pr[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) { xv[u] = nx[u]; yv[u] = ny[u]; }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// products precomputed (independent work), then chain over products via LDS.128
template <int U>
__global__ void v2_prod_then_chain(double* out, long long* cyc, int reps) {
    __shared__ double tile[2][T * P];
    __shared__ __align__(16) double prod[64][T + 2];
    for (int i = threadIdx.x; i < T * P; i += blockDim.x) { tile[0][i] = 1.0 + i * 1e-3; tile[1][i] = 0.5 - i * 1e-4; }
    __syncthreads();
    const double* xs = tile[0] + (threadIdx.x & 7);
    const double* ys = tile[1] + (threadIdx.x >> 3);
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int k = 0; k < T; ++k) prod[threadIdx.x][k] = __dmul_rn(xs[k * P], ys[k * P]);
        __syncwarp();
        const double2* pp = reinterpret_cast<const double2*>(prod[threadIdx.x]);
#pragma unroll 1
        for (int kb = 0; kb < T / 2; kb += U) {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = pp[kb + u];
#pragma unroll
            for (int u = 0; u < U; ++u) { acc = __dadd_rn(acc, v[u].x); acc = __dadd_rn(acc, v[u].y); }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// pure register chain (lower bound)
__global__ void v3_regs(double* out, long long* cyc, int reps) {
    double acc = 0.0, x = 1.0 + threadIdx.x * 1e-3, y = 0.5;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 16
        for (int k = 0; k < T; ++k) acc = __dadd_rn(acc, __dmul_rn(x + k, y));
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&cyc, 8);
    const int reps = 256;
    auto report = [&](const char* name) {
        cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("%-28s %6.2f cycles/step\n", name, (double)h / (reps * T));
    };
    for (int w = 0; w < 2; ++w) {
        v0_naive<<<1, 64>>>(out, cyc, reps); report("v0 naive (unroll 16)");
        v1_batched<8><<<1, 64>>>(out, cyc, reps); report("v1 batched U=8");
        v1_batched<16><<<1, 64>>>(out, cyc, reps); report("v1 batched U=16");
        v2_prod_then_chain<4><<<1, 64>>>(out, cyc, reps); report("v2 products then chain");
        v3_regs<<<1, 64>>>(out, cyc, reps); report("v3 register-only chain");
    }
    return 0;
}
