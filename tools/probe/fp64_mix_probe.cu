// FP64 issue mix probe (round 2): what does a dependent DADD chain cost per
// step when each step also issues a DMUL (or DFMA) and shared loads?  One warp,
// clock64 around a long unrolled loop; every variant keeps its results live.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix_probe fp64_mix_probe.cu
#include <cstdio>

constexpr int N = 4096;  // steps per timed loop (unrolled by 16)

template <int MODE>
__global__ void mix(const double* __restrict__ in, double* __restrict__ out, long long* cyc) {
    __shared__ double sh[4096 + 64];
    for (int i = threadIdx.x; i < 4096 + 64; i += blockDim.x) sh[i] = in[i % 64] + i * 1e-9;
    __syncthreads();
    double acc = 0.0, acc2 = 0.0, x = in[threadIdx.x % 8], y = in[8 + threadIdx.x % 8];
    double p[16], q[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        p[u] = in[16 + u];
        q[u] = in[32 + u];
    }
    const double* s = sh + (threadIdx.x & 7);
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < N; k += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (MODE == 0) {  // DADD chain, register addend
                acc = __dadd_rn(acc, p[u]);
            } else if (MODE == 1) {  // + an independent DMUL per step (its own chains)
                acc = __dadd_rn(acc, p[u]);
                q[u] = __dmul_rn(q[u], x);
            } else if (MODE == 2) {  // + an independent DFMA per step
                acc = __dadd_rn(acc, p[u]);
                q[u] = fma(q[u], x, y);
            } else if (MODE == 3) {  // + an independent DADD per step
                acc = __dadd_rn(acc, p[u]);
                q[u] = __dadd_rn(q[u], x);
            } else if (MODE == 4) {  // two independent DADD chains
                acc = __dadd_rn(acc, p[u]);
                acc2 = __dadd_rn(acc2, q[u]);
            } else if (MODE == 5) {  // chain + 1 LDS per step (addend from smem, 16 steps ahead)
                acc = __dadd_rn(acc, p[u]);
                p[u] = s[(k + u) * 8 % 4096];
            } else if (MODE == 6) {  // chain + DMUL + 1 LDS (the transposed chain kernel's step)
                acc = __dadd_rn(acc, p[u]);
                p[u] = __dmul_rn(q[u], y);
                q[u] = s[(k + u) * 8 % 4096];
            } else if (MODE == 7) {  // chain + DFMA(a, b, -0) product + 1 LDS
                acc = __dadd_rn(acc, p[u]);
                p[u] = fma(q[u], y, -0.0);
                q[u] = s[(k + u) * 8 % 4096];
            } else if (MODE == 8) {  // pure DMUL chain (dependent)
                acc = __dmul_rn(acc + 1.0, p[u]);
            } else if (MODE == 9) {  // pure DFMA chain
                acc = fma(acc, p[u], q[u]);
            }
        }
    }
    long long t1 = clock64();
    double r = acc + acc2;
#pragma unroll
    for (int u = 0; u < 16; ++u) r += p[u] + q[u];
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name, const double* in, double* out, long long* cyc) {
    long long h = 0;
    for (int rep = 0; rep < 3; ++rep) {
        mix<MODE><<<1, 32>>>(in, out, cyc);
        cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    }
    printf("mode %d %-52s %6.2f cycles/step\n", MODE, name, (double)h / N);
}

int main() {
    double* in;
    double* out;
    long long* cyc;
    cudaMalloc(&in, 64 * sizeof(double));
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    double h[64];
    for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 1e-3;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    run<0>("DADD chain (register addend)", in, out, cyc);
    run<1>("DADD chain + independent DMUL", in, out, cyc);
    run<2>("DADD chain + independent DFMA", in, out, cyc);
    run<3>("DADD chain + independent DADD", in, out, cyc);
    run<4>("two DADD chains", in, out, cyc);
    run<5>("DADD chain + LDS", in, out, cyc);
    run<6>("DADD chain + DMUL + LDS (product 16 steps ahead)", in, out, cyc);
    run<7>("DADD chain + DFMA(a,b,-0) + LDS", in, out, cyc);
    run<8>("dependent DMUL(+DADD) chain", in, out, cyc);
    run<9>("dependent DFMA chain", in, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
