// Shared-memory load latency on B200 (round 2): dependent LDS.64 / LDS.128
// chains (pointer chasing), one warp, and the same under a second warp doing
// streaming loads.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_lat_probe lds_lat_probe.cu
#include <cstdio>
template <int W128>
__global__ void lat(long long* cyc, int* sink) {
    __shared__ __align__(16) long long idx[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) idx[i] = (i * 37 + 64) & 4095 & ~1;
    __syncthreads();
    if (threadIdx.x >= 32) {  // background streaming warps
        long long s = 0;
        for (int r = 0; r < 64; ++r)
            for (int i = threadIdx.x; i < 4096; i += blockDim.x - 32) s += idx[i];
        if (s == 12345) sink[1] = 1;
        return;
    }
    int j = threadIdx.x * 2;
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < 1024; ++k) {
        if (W128) {
            longlong2 v = *reinterpret_cast<const longlong2*>(&idx[j]);
            j = (int)(v.x + (v.y & 0));
        } else {
            j = (int)idx[j];
        }
    }
    long long t1 = clock64();
    if (j == -1) sink[0] = j;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    long long* cyc; int* sink; long long h;
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 8);
    for (int th : {32, 64, 128}) {
        lat<0><<<1, th>>>(cyc, sink); lat<0><<<1, th>>>(cyc, sink);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("LDS.64  dependent, %3d threads: %.1f cycles/load (incl. ~2 cycles of loop)\n", th, h / 1024.0);
        lat<1><<<1, th>>>(cyc, sink); lat<1><<<1, th>>>(cyc, sink);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("LDS.128 dependent, %3d threads: %.1f cycles/load\n", th, h / 1024.0);
    }
    return 0;
}
