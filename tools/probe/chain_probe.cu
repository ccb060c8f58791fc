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

// products precomputed in shared memory, [k][chain] layout; DADD-only chain
template <int U>
__global__ void v4_prod_smem(double* out, long long* cyc, int reps) {
    __shared__ double prod[T][64];
    for (int i = threadIdx.x; i < T * 64; i += blockDim.x) prod[i / 64][i % 64] = 1.0 + i * 1e-3;
    __syncthreads();
    const double* ps = &prod[0][threadIdx.x];
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ps[u * 64];
#pragma unroll 1
        for (int kb = 0; kb < T; kb += U) {
            const int kn = (kb + U < T) ? kb + U : 0;
            double nv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) nv[u] = ps[(kn + u) * 64];
#pragma unroll
            for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, v[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = nv[u];
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// in-thread products, software-pipelined: iteration b adds batch b's products
// (computed in iteration b-1, loop-carried) while forming batch b+1's products
// and loading batch b+2's operands.
template <int U>
__global__ void v5_pipelined(double* out, long long* cyc, int reps) {
    __shared__ double tile[2][T * P];
    for (int i = threadIdx.x; i < T * P; i += blockDim.x) { tile[0][i] = 1.0 + i * 1e-3; tile[1][i] = 0.5 - i * 1e-4; }
    __syncthreads();
    const double* xs = tile[0] + (threadIdx.x & 7);
    const double* ys = tile[1] + (threadIdx.x >> 3);
    double acc = 0.0;
    constexpr int NB = T / U;
    const int nb = reps * NB;
    double pr[U], xv[U], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(xs[u * P], ys[u * P]);
#pragma unroll
    for (int u = 0; u < U; ++u) { xv[u] = xs[((U + u) % T) * P]; yv[u] = ys[((U + u) % T) * P]; }
    long long t0 = clock64();
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
        const int k2 = ((b + 2) % NB) * U;
        double npr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc = __dadd_rn(acc, pr[u]);
            npr[u] = __dmul_rn(xv[u], yv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { xv[u] = xs[(k2 + u) * P]; yv[u] = ys[(k2 + u) * P]; }
#pragma unroll
        for (int u = 0; u < U; ++u) pr[u] = npr[u];
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
        v5_pipelined<8><<<1, 64>>>(out, cyc, reps); report("v5 pipelined U=8");
        v5_pipelined<16><<<1, 64>>>(out, cyc, reps); report("v5 pipelined U=16");
        v5_pipelined<32><<<1, 64>>>(out, cyc, reps); report("v5 pipelined U=32");
        v4_prod_smem<8><<<1, 64>>>(out, cyc, reps); report("v4 smem products U=8");
        v4_prod_smem<16><<<1, 64>>>(out, cyc, reps); report("v4 smem products U=16");
        v4_prod_smem<32><<<1, 64>>>(out, cyc, reps); report("v4 smem products U=32");
    }
    return 0;
}
