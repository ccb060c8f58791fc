// Chains per thread (C = 1, 2, 4): the production chain_kernel runs one
// sequential dot-product chain per thread; here each thread runs C
// independent chains interleaved in program order so that each chain's
// dependent DADD has the other chains' DMUL / LDS in its latency shadow.
// Checks the results bit for bit against the production kernel and times
// both (P = 8, the gram-phase chain set, n = 16384).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o chain_multi_probe chain_multi_probe.cu
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "exact_kernels.cuh"

using namespace coopcg_gpu;

template <int P, int T, int S, int C, int U, int W, int FENCE = 0>
__global__ void __launch_bounds__(32 * (1 + W))
    chainC_kernel(const double* __restrict__ s0, const double* __restrict__ s1, const double* __restrict__ s2,
                  int nsrc, int n, const ChainDesc* __restrict__ descs, int nchains, double* __restrict__ out) {
    static_assert(T % (2 * U) == 0, "tile rows must be an even number of batches");
    constexpr int NBT = T / U;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* buf = reinterpret_cast<double*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(buf + static_cast<size_t>(S) * nsrc * T * P);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntiles = (n + T - 1) / T;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int rows = min(T, n - t * T);
                const uint32_t bytes = static_cast<uint32_t>(rows) * P * 8u;
                mbar_arrive_expect_tx(&full[s], bytes * nsrc);
                double* dst = buf + static_cast<size_t>(s) * nsrc * T * P;
                bulk_g2s(dst, s0 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 1) bulk_g2s(dst + T * P, s1 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 2) bulk_g2s(dst + 2 * T * P, s2 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    // thread t of the grid runs chains t, t + nthr, ..., (C of them)
    const int nthr = gridDim.x * W * 32;
    const int t0 = blockIdx.x * (W * 32) + (tid - 32);
    int xoff[C], yoff[C];
    bool live[C];
    ChainDesc d[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int ci = t0 + c * nthr;
        live[c] = ci < nchains;
        d[c] = live[c] ? descs[ci] : ChainDesc{0, 0, 0, 0, 0, 0, 0};
        xoff[c] = d[c].sx * T * P + d[c].a;
        yoff[c] = d[c].sy * T * P + d[c].b;
    }
    const int nb = (n + U - 1) / U;
    auto tile_wait = [&](int t) {
        if (t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    auto batch_base = [&](int j) -> const double* {
        return buf + static_cast<size_t>((j / NBT) % S) * nsrc * T * P + (j % NBT) * U * P;
    };
    double acc[C];
    double pr[C][U], xe[C][U], ye[C][U], xo[C][U], yo[C][U];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    auto step = [&](int b, const double (&xr)[C][U], const double (&yr)[C][U], double (&xw)[C][U],
                    double (&yw)[C][U]) {
        const double* b2 = batch_base(b + 2);
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], pr[c][u]);
#pragma unroll
            for (int c = 0; c < C; ++c) pr[c][u] = __dmul_rn(xr[c][u], yr[c][u]);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                xw[c][u] = b2[xoff[c] + u * P];
                yw[c][u] = b2[yoff[c] + u * P];
            }
        }
        // FENCE: a never-taken branch on an opaque value ends the basic block,
        // so the scheduler cannot sink this batch's DMULs next to the DADDs
        // of the next step that consume them
        if (FENCE && nsrc > 1000) __trap();
    };
    tile_wait(0);
    {
        const double* b0 = batch_base(0);
        const double* b1 = batch_base(1);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                pr[c][u] = __dmul_rn(b0[xoff[c] + u * P], b0[yoff[c] + u * P]);
                xo[c][u] = b1[xoff[c] + u * P];
                yo[c][u] = b1[yoff[c] + u * P];
            }
    }
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
        tile_wait(t + 1);
        const int b0 = t * NBT;
        if ((t + 1) * T <= n) {
#pragma unroll
            for (int q = 0; q < NBT; q += 2) {
                step(b0 + q, xo, yo, xe, ye);
                step(b0 + q + 1, xe, ye, xo, yo);
            }
        } else {
            for (int q = 0; q < NBT && b0 + q < nb; ++q) {
                const int b = b0 + q;
                if (b == nb - 1) {
                    const int rem = n - b * U;
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int c = 0; c < C; ++c)
                            if (u < rem) acc[c] = __dadd_rn(acc[c], pr[c][u]);
                } else if (q & 1) {
                    step(b, xe, ye, xo, yo);
                } else {
                    step(b, xo, yo, xe, ye);
                }
            }
        }
        __syncwarp();
        mbar_arrive_lane0(&empty[t % S], lane);
    }
#pragma unroll
    for (int c = 0; c < C; ++c)
        if (live[c]) out[d[c].out] = d[c].neg ? -acc[c] : acc[c];
}

template <class K>
float timeit(K launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return ms / 10 * 1e3f;
}

template <int P, int T, int S, int C, int U, int W>
void variant(const double* s0, const double* s1, const double* s2, int n, const ChainDesc* d, int nch,
             double* out, const std::vector<double>& ref, const char* name) {
    auto k = chainC_kernel<P, T, S, C, U, W>;
    size_t smem = chain_smem_bytes(P, T, S, 3);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int per_cta = W * 32 * C;
    const int grid = (nch + per_cta - 1) / per_cta;
    cudaMemset(out, 0, 8192 * 8);
    const float us = timeit([&] { k<<<grid, 32 * (1 + W), smem>>>(s0, s1, s2, 3, n, d, nch, out); });
    std::vector<double> got(8192);
    cudaMemcpy(got.data(), out, 8192 * 8, cudaMemcpyDeviceToHost);
    const bool same = std::memcmp(got.data(), ref.data(), 8192 * 8) == 0;
    std::printf("%-34s T=%3d S=%d C=%d U=%2d W=%d grid=%d : %7.1f us = %5.2f cycles/step  %s\n", name, T, S, C, U, W,
                grid, us, us * 1.965e3 / n, same ? "bit-identical" : "MISMATCH");
}

template <int P, int T, int S, int C, int U, int W, int F>
void variant2(const double* s0, const double* s1, const double* s2, int n, const ChainDesc* d, int nch,
              double* out, const std::vector<double>& ref, const char* name) {
    auto k = chainC_kernel<P, T, S, C, U, W, F>;
    size_t smem = chain_smem_bytes(P, T, S, 3);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int per_cta = W * 32 * C;
    const int grid = (nch + per_cta - 1) / per_cta;
    cudaMemset(out, 0, 8192 * 8);
    const float us = timeit([&] { k<<<grid, 32 * (1 + W), smem>>>(s0, s1, s2, 3, n, d, nch, out); });
    std::vector<double> got(8192);
    cudaMemcpy(got.data(), out, 8192 * 8, cudaMemcpyDeviceToHost);
    const bool same = std::memcmp(got.data(), ref.data(), 8192 * 8) == 0;
    std::printf("%-34s T=%3d S=%d C=%d U=%2d W=%d grid=%d : %7.1f us = %5.2f cycles/step  %s\n", name, T, S, C, U, W,
                grid, us, us * 1.965e3 / n, same ? "bit-identical" : "MISMATCH");
}

int main() {
    constexpr int P = 8;
    const int n = 16384, p = 8;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1);
    std::vector<double> h0((size_t)n * P), h1((size_t)n * P), h2((size_t)n * P);
    for (auto* v : {&h0, &h1, &h2})
        for (auto& x : *v) x = U(rng);
    double *s0, *s1, *s2, *out;
    cudaMalloc(&s0, (size_t)n * P * 8);
    cudaMalloc(&s1, (size_t)n * P * 8);
    cudaMalloc(&s2, (size_t)n * P * 8);
    cudaMalloc(&out, 8192 * 8);
    cudaMemcpy(s0, h0.data(), h0.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(s1, h1.data(), h1.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(s2, h2.data(), h2.size() * 8, cudaMemcpyHostToDevice);
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
    // production kernel (reference output + time)
    std::vector<double> ref(8192);
    {
        auto k = chain_kernel<P, 384, 3>;
        size_t smem = chain_smem_bytes(P, 384, 3, 3);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaMemset(out, 0, 8192 * 8);
        const float us = timeit([&] { k<<<(nch + 63) / 64, kChainThreads, smem>>>(s0, s1, s2, 3, n, d, nch, out, nullptr); });
        cudaMemcpy(ref.data(), out, 8192 * 8, cudaMemcpyDeviceToHost);
        std::printf("%-34s T=384 S=3 C=1 U=16 W=2 : %7.1f us = %5.2f cycles/step\n", "production chain_kernel", us,
                    us * 1.965e3 / n);
    }
    variant<P, 384, 3, 1, 16, 2>(s0, s1, s2, n, d, nch, out, ref, "C=1 (production shape)");
    variant<P, 384, 3, 1, 16, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=16 W=1");
    variant<P, 384, 3, 1, 8, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=8 W=1");
    variant2<P, 384, 3, 1, 16, 1, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=16 W=1 FENCE");
    variant<P, 192, 4, 1, 16, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=16 W=1 T=192 S=4");
    variant2<P, 384, 3, 1, 16, 2, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=16 FENCE");
    variant2<P, 384, 3, 1, 8, 2, 1>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=8 FENCE");
    variant2<P, 384, 3, 2, 8, 2, 1>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=8 FENCE");
    variant<P, 384, 3, 1, 8, 2>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=8");
    variant<P, 384, 3, 2, 8, 2>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=8 W=2");
    variant<P, 384, 3, 2, 8, 1>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=8 W=1");
    variant<P, 384, 3, 2, 8, 4>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=8 W=4");
    variant<P, 384, 3, 2, 12, 2>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=12 W=2");
    variant<P, 384, 3, 3, 8, 2>(s0, s1, s2, n, d, nch, out, ref, "C=3 U=8 W=2");
    variant<P, 384, 3, 4, 4, 2>(s0, s1, s2, n, d, nch, out, ref, "C=4 U=4 W=2");
    variant<P, 384, 3, 4, 8, 2>(s0, s1, s2, n, d, nch, out, ref, "C=4 U=8 W=2");
    variant<P, 384, 3, 2, 8, 3>(s0, s1, s2, n, d, nch, out, ref, "C=2 U=8 W=3");
    variant<P, 384, 3, 1, 16, 4>(s0, s1, s2, n, d, nch, out, ref, "C=1 U=16 W=4");
    std::printf("(DADD dependent latency 8.76 cycles: %.1f us per 16384-step chain)\n", n * 8.76 / 1.965e3);
    return 0;
}
