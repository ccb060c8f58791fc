// Throughput of cp.async.bulk (1-D TMA) global->shared for one CTA and for a
// full grid, as a function of copy size and pipeline depth; versus cp.async
// (LDGSTS) 16-byte copies by all threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o bulk_probe bulk_probe.cu
#include <cstdio>
#include "common.cuh"

using namespace coopcg_gpu;

// Each CTA streams `total` bytes from src (its own slice) through S stages of `chunk` bytes.
__global__ void bulk_stream(const char* src, size_t per_cta, int chunk, int S, double* sink, int copies_per_stage) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)S * chunk);
    const char* base = src + (size_t)blockIdx.x * per_cta;
    const int ntiles = (int)(per_cta / chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int t) {
        const int s = t % S;
        mbar_arrive_expect_tx(&bar[s], chunk);
        const int part = chunk / copies_per_stage;
        for (int c = 0; c < copies_per_stage; ++c)
            bulk_g2s(smem + (size_t)s * chunk + c * part, base + (size_t)t * chunk + c * part, part, &bar[s]);
    };
    if (threadIdx.x == 0)
        for (int t = 0; t < S - 1 && t < ntiles; ++t) issue(t);
    double acc = 0;
    for (int t = 0; t < ntiles; ++t) {
        if (threadIdx.x == 0 && t + S - 1 < ntiles) issue(t + S - 1);
        mbar_wait(&bar[t % S], (t / S) & 1);
        acc += reinterpret_cast<const double*>(smem + (size_t)(t % S) * chunk)[threadIdx.x];
        __syncthreads();
    }
    if (acc == 1234.5) sink[0] = acc;
}

int main() {
    size_t bytes = (size_t)2 << 30;
    char* src;
    double* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(src, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int ctas, chunk, S, cps; };
    Cfg cfgs[] = {
        {1, 4096, 6, 1}, {1, 16384, 4, 1}, {1, 65536, 2, 1}, {1, 16384, 4, 32},
        {148, 4096, 6, 1}, {148, 16384, 4, 1}, {148, 32768, 4, 1}, {148, 16384, 4, 32},
        {296, 16384, 4, 1}, {444, 16384, 4, 1}, {296, 32768, 3, 1},
    };
    for (auto c : cfgs) {
        size_t per_cta = (c.ctas == 1) ? (size_t)64 << 20 : (bytes / c.ctas) / c.chunk * c.chunk;
        size_t smem = (size_t)c.S * c.chunk + c.S * 8;
        cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        bulk_stream<<<c.ctas, 128, smem>>>(src, per_cta, c.chunk, c.S, sink, c.cps);
        cudaEventRecord(e0);
        bulk_stream<<<c.ctas, 128, smem>>>(src, per_cta, c.chunk, c.S, sink, c.cps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t e = cudaGetLastError();
        double tot = (double)per_cta * c.ctas;
        std::printf("ctas=%4d chunk=%6d S=%d copies/stage=%2d : %8.1f GB/s total, %7.2f GB/s per CTA, %.3f us per stage %s\n",
                    c.ctas, c.chunk, c.S, c.cps, tot / (ms * 1e-3) / 1e9, tot / c.ctas / (ms * 1e-3) / 1e9,
                    ms * 1e3 / (per_cta / c.chunk), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
