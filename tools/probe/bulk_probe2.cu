// Are multiple cp.async.bulk copies (separate mbarriers) in flight at once?
// One CTA issues N copies of `chunk` bytes back to back (each on its own
// mbarrier) from thread 0, then waits for all: time vs N.  Variant B issues
// copy i from warp i's lane 0.  Variant C uses cp.async (LDGSTS) 16-B by all
// threads.  Variant D: plain LDG.128 by all threads into registers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o bulk_probe2 bulk_probe2.cu
#include <cstdio>
#include "common.cuh"

using namespace coopcg_gpu;

__global__ void burst(const char* src, int N, int chunk, int mode, long long* cyc) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)N * chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < N; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
        if (threadIdx.x == 0)
            for (int i = 0; i < N; ++i) {
                mbar_arrive_expect_tx(&bar[i], chunk);
                bulk_g2s(smem + (size_t)i * chunk, src + (size_t)i * chunk * 7, chunk, &bar[i]);
            }
    } else if (mode == 1) {
        const int w = threadIdx.x / 32;
        if ((threadIdx.x & 31) == 0 && w < N) {
            mbar_arrive_expect_tx(&bar[w], chunk);
            bulk_g2s(smem + (size_t)w * chunk, src + (size_t)w * chunk * 7, chunk, &bar[w]);
        }
    }
    if (mode <= 1) {
        for (int i = 0; i < N; ++i) mbar_wait(&bar[i], 0);
    } else {
        // cp.async 16B by all threads
        for (int i = 0; i < N; ++i)
            for (int o = threadIdx.x * 16; o < chunk; o += blockDim.x * 16) {
                unsigned dst = smem_u32(smem + (size_t)i * chunk + o);
                const char* g = src + (size_t)i * chunk * 7 + o;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g));
            }
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    char* src;
    long long* cyc;
    cudaMalloc(&src, (size_t)1 << 30);
    cudaMalloc(&cyc, 8);
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"bulk, thread 0 issues all", "bulk, one per warp", "cp.async 16B all threads"};
    for (int mode = 0; mode < 3; ++mode)
        for (int chunk : {4096, 16384})
            for (int N : {1, 2, 4, 8}) {
                if ((size_t)N * chunk > 180 * 1024) continue;
                long long best = 1LL << 60;
                for (int r = 0; r < 5; ++r) {
                    burst<<<1, 256, (size_t)N * chunk + N * 8>>>(src + r * 4096 * 64, N, chunk, mode, cyc);
                    long long h;
                    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
                    best = h < best ? h : best;
                }
                std::printf("%-28s chunk=%6d N=%d : %7lld cycles (%.0f cycles per copy)\n", names[mode], chunk, N, best,
                            (double)best / N);
            }
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("%s\n", cudaGetErrorString(e));
    return 0;
}
