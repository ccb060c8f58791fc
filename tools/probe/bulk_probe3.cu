// Streaming ring variants for cp.async.bulk: which loop structure keeps
// S-1 copies in flight?  One CTA (and a full grid), 16 KB stages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o bulk_probe3 bulk_probe3.cu
#include <cstdio>
#include "common.cuh"

using namespace coopcg_gpu;

__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// mode 0: thread 0 produces + consumes, __syncthreads per stage (current design)
// mode 1: same with polling test_wait
// mode 2: warp 0 = producer only (waits on per-stage empty barriers), warps 1.. consume
template <int S>
__global__ void stream(const char* src, size_t per_cta, int chunk, int mode, double* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * chunk);
    uint64_t* empty = full + S;
    const char* base = src + (size_t)blockIdx.x * per_cta;
    const int ntiles = (int)(per_cta / chunk);
    const int nconsumers = (mode == 2) ? (blockDim.x / 32 - 1) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nconsumers > 0 ? nconsumers : 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    double acc = 0;
    if (mode <= 1) {
        auto issue = [&](int t) {
            const int s = t % S;
            mbar_arrive_expect_tx(&full[s], chunk);
            bulk_g2s(smem + (size_t)s * chunk, base + (size_t)t * chunk, chunk, &full[s]);
        };
        if (threadIdx.x == 0)
            for (int t = 0; t < S - 1 && t < ntiles; ++t) issue(t);
        for (int t = 0; t < ntiles; ++t) {
            if (threadIdx.x == 0 && t + S - 1 < ntiles) issue(t + S - 1);
            if (mode == 0) mbar_wait(&full[t % S], (t / S) & 1);
            else mbar_wait_poll(&full[t % S], (t / S) & 1);
            acc += reinterpret_cast<const double*>(smem + (size_t)(t % S) * chunk)[threadIdx.x];
            __syncthreads();
        }
    } else {
        const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
        if (warp == 0) {
            if (lane == 0)
                for (int t = 0; t < ntiles; ++t) {
                    const int s = t % S;
                    if (t >= S) mbar_wait(&empty[s], ((t / S) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], chunk);
                    bulk_g2s(smem + (size_t)s * chunk, base + (size_t)t * chunk, chunk, &full[s]);
                }
        } else {
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % S;
                mbar_wait(&full[s], (t / S) & 1);
                acc += reinterpret_cast<const double*>(smem + (size_t)s * chunk)[threadIdx.x];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
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
    const int chunk = 16384, S = 4;
    cudaFuncSetAttribute(stream<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * chunk + 64);
    const char* names[] = {"produce+consume, try_wait", "produce+consume, test_wait poll", "warp-specialized producer"};
    for (int ctas : {1, 148, 296})
        for (int mode = 0; mode < 3; ++mode) {
            size_t per_cta = (ctas == 1) ? (size_t)64 << 20 : (bytes / ctas) / chunk * chunk;
            stream<S><<<ctas, 128, S * chunk + 64>>>(src, per_cta, chunk, mode, sink);
            cudaEventRecord(e0);
            stream<S><<<ctas, 128, S * chunk + 64>>>(src, per_cta, chunk, mode, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double tot = (double)per_cta * ctas;
            std::printf("ctas=%3d %-34s %8.1f GB/s total %7.2f GB/s/CTA  %.3f us/stage  %s\n", ctas, names[mode],
                        tot / (ms * 1e-3) / 1e9, tot / ctas / (ms * 1e-3) / 1e9, ms * 1e3 / (per_cta / chunk),
                        cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
