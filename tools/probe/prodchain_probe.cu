// Exact sequential chains over PRECOMPUTED products (acc = acc + prod[k], k
// ascending): each chain thread streams its own contiguous product array
// (L2-resident) through a register prefetch ring.  Measures us per chain phase
// at n = 16384 for 136 chains (the p = 8 gram phase), vs the ~9-cycle DADD floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o prodchain_probe prodchain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// products stored [k][chain] (ld = padded chain count): a warp's step is one
// coalesced 256-byte load.
template <int DEPTH>
__global__ void prodchain_km(const double* __restrict__ prod, int n, int ld, int nchains, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchains) return;
    const double* src = prod + c;
    double ring[DEPTH];
#pragma unroll
    for (int i = 0; i < DEPTH; ++i) ring[i] = src[static_cast<size_t>(i) * ld];
    double acc = 0.0;
    int base = 0;
    for (; base + 2 * DEPTH <= n; base += DEPTH) {
#pragma unroll
        for (int i = 0; i < DEPTH; ++i) {
            const double v = ring[i];
            ring[i] = __ldcg(src + static_cast<size_t>(base + DEPTH + i) * ld);
            acc = __dadd_rn(acc, v);
        }
    }
#pragma unroll
    for (int i = 0; i < DEPTH; ++i) acc = __dadd_rn(acc, ring[i]);
    for (int k = base + DEPTH; k < n; ++k) acc = __dadd_rn(acc, src[static_cast<size_t>(k) * ld]);
    out[c] = acc;
}

template <int DEPTH>
__global__ void prodchain(const double* __restrict__ prod, int n, int nchains, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchains) return;
    const double2* src = reinterpret_cast<const double2*>(prod + static_cast<size_t>(c) * n);
    const int m = n / 2;
    double2 ring[DEPTH];
#pragma unroll
    for (int i = 0; i < DEPTH; ++i) ring[i] = src[i];
    double acc = 0.0;
    int base = 0;
    for (; base + 2 * DEPTH <= m; base += DEPTH) {
#pragma unroll
        for (int i = 0; i < DEPTH; ++i) {
            const double2 v = ring[i];
            ring[i] = __ldcg(src + base + DEPTH + i);
            acc = __dadd_rn(acc, v.x);
            acc = __dadd_rn(acc, v.y);
        }
    }
    // drain: ring holds [base, base + DEPTH)
#pragma unroll
    for (int i = 0; i < DEPTH; ++i) {
        acc = __dadd_rn(acc, ring[i].x);
        acc = __dadd_rn(acc, ring[i].y);
    }
    for (int k = base + DEPTH; k < m; ++k) {
        const double2 v = src[k];
        acc = __dadd_rn(acc, v.x);
        acc = __dadd_rn(acc, v.y);
    }
    out[c] = acc;
}

template <int DEPTH>
float run(const double* prod, int n, int nch, double* out, int tpb) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    prodchain<DEPTH><<<(nch + tpb - 1) / tpb, tpb>>>(prod, n, nch, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) prodchain<DEPTH><<<(nch + tpb - 1) / tpb, tpb>>>(prod, n, nch, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10 * 1e3f;
}

template <int DEPTH>
float run_km(const double* prod, int n, int nch, double* out, int tpb) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int ld = (nch + 31) / 32 * 32;
    prodchain_km<DEPTH><<<(nch + tpb - 1) / tpb, tpb>>>(prod, n, ld, nch, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) prodchain_km<DEPTH><<<(nch + tpb - 1) / tpb, tpb>>>(prod, n, ld, nch, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10 * 1e3f;
}

int main() {
    const int n = 16384, nch = 136;
    double *prod, *out;
    cudaMalloc(&prod, (size_t)n * nch * 8);
    cudaMalloc(&out, nch * 8);
    cudaMemset(prod, 0, (size_t)n * nch * 8);
    for (int tpb : {32, 64}) {
        std::printf("[k][chain] tpb=%d depth=16 : %7.1f us\n", tpb, run_km<16>(prod, n, nch, out, tpb));
        std::printf("[k][chain] tpb=%d depth=32 : %7.1f us\n", tpb, run_km<32>(prod, n, nch, out, tpb));
        std::printf("[k][chain] tpb=%d depth=64 : %7.1f us\n", tpb, run_km<64>(prod, n, nch, out, tpb));
        std::printf("[k][chain] tpb=%d depth=96 : %7.1f us\n", tpb, run_km<96>(prod, n, nch, out, tpb));
    }
    for (int tpb : {32}) {
        std::printf("tpb=%d depth=8  : %7.1f us\n", tpb, run<8>(prod, n, nch, out, tpb));
        std::printf("tpb=%d depth=16 : %7.1f us\n", tpb, run<16>(prod, n, nch, out, tpb));
        std::printf("tpb=%d depth=32 : %7.1f us\n", tpb, run<32>(prod, n, nch, out, tpb));
        std::printf("tpb=%d depth=48 : %7.1f us\n", tpb, run<48>(prod, n, nch, out, tpb));
    }
    std::printf("floor at 9 cycles/step, 1.9 GHz: %.1f us; %s\n", n * 9 / 1.9e3,
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
