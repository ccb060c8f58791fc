// L2 residency probe: stream a buffer repeatedly with cp.async.bulk, the first
// fraction f of every CTA slice copied with an L2 evict_last policy, the rest
// evict_first.  Question: how much of a re-streamed A (cfg 1: 134 MB, cfg 2:
// 2.15 GB) can stay in the 126 MB L2 across passes, and what does a pass cost?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o l2res_probe l2res_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace coopcg_gpu;

__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t pol_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

constexpr int S = 4;
constexpr int CHUNK = 32768;

__global__ void stream(const char* src, size_t per_cta, size_t res_bytes, int mode, double* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * CHUNK);
    uint64_t* empty = full + S;
    const char* base = src + (size_t)blockIdx.x * per_cta;
    const int ntiles = (int)(per_cta / CHUNK);
    const int nconsumers = blockDim.x / 32 - 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nconsumers);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pf = l2_evict_first_policy();
            const uint64_t pl = mode == 2 ? pol_evict_normal() : pol_evict_last();
            for (int t = 0; t < ntiles; ++t) {
                const int s = t % S;
                if (t >= S) mbar_wait(&empty[s], ((t / S) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], CHUNK);
                const bool res = (size_t)t * CHUNK < res_bytes;
                bulk_g2s_evict_first(smem + (size_t)s * CHUNK, base + (size_t)t * CHUNK, CHUNK, &full[s],
                                     res ? pl : pf);
            }
        }
        return;
    }
    double acc = 0;
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % S;
        mbar_wait(&full[s], (t / S) & 1);
        acc += reinterpret_cast<const double*>(smem + (size_t)s * CHUNK)[threadIdx.x - 32];
        __syncwarp();
        mbar_arrive_lane0(&empty[s], lane);
    }
    if (acc == 12345.0) sink[0] = acc;
}

__global__ void flush(double* buf, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = (double)i;
}

int main(int argc, char** argv) {
    int dev = 0;
    cudaSetDevice(dev);
    int sms = 0, l2 = 0, maxp = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    printf("SMs %d  L2 %.1f MB  max persisting %.1f MB\n", sms, l2 / 1e6, maxp / 1e6);
    const size_t sizes[] = {(size_t)4096 * 4096 * 8, (size_t)16384 * 16384 * 8};
    char* buf;
    cudaMalloc(&buf, sizes[1] + (1 << 20));
    cudaMemset(buf, 1, sizes[1]);
    double* fl;
    cudaMalloc(&fl, (size_t)256 << 20);
    double* sink;
    cudaMalloc(&sink, 8);
    const size_t smem = (size_t)S * CHUNK + 2 * S * 8;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int setaside = 0; setaside < 2; ++setaside) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside ? (size_t)maxp : 0);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
        for (size_t total : sizes) {
            const int ctas = sms;
            size_t per_cta = (total / ctas) / CHUNK * CHUNK;
            for (int mode = 1; mode <= 2; ++mode) {
                for (double mb : {0.0, 32.0, 48.0, 64.0, 80.0, 96.0, 112.0, 128.0}) {
                    if (mode == 2 && mb != 0.0 && mb != 96.0) continue;
                    size_t res = (size_t)(mb * 1e6 / ctas);
                    flush<<<1184, 256>>>(fl, ((size_t)256 << 20) / 8);
                    for (int w = 0; w < 3; ++w) stream<<<ctas, 160, smem>>>(buf, per_cta, res, mode, sink);
                    const int reps = total > (1u << 30) ? 10 : 50;
                    cudaEventRecord(e0);
                    for (int r = 0; r < reps; ++r) stream<<<ctas, 160, smem>>>(buf, per_cta, res, mode, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double us = ms * 1e3 / reps;
                    printf("setaside %6.1f MB  total %7.1f MB  %s  resident %5.1f MB  %8.2f us/pass  %7.1f GB/s eff\n",
                           got / 1e6, ctas * per_cta / 1e6, mode == 1 ? "evict_last  " : "evict_normal", mb, us,
                           ctas * per_cta / (us * 1e3));
                }
            }
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
