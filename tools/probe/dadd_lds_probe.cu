// dadd_lds_probe.cu -- why do DADD chains fed from shared memory run slowly?
// One warp; chain acc += v[k] over 4096 steps, v from (a) registers,
// (b) LDS 16 ahead (batch), (c) LDS.128 batch, (d) DMUL of LDS operands,
// (e) batch LDS with a __syncwarp between batches, (f) batch LDS after a
// named-barrier handshake with a second warp that only arrives.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096, U = 16;

template <int V>
__global__ void k(double* out, long long* cyc) {
    __shared__ double sm[N + 64];
    for (int i = threadIdx.x; i < N + 64; i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
    __syncthreads();
    if (V == 5 && threadIdx.x >= 32) {  // partner warp: arrive per batch
        for (int b = 0; b < N / U; ++b) asm volatile("bar.sync 1, 64;" ::: "memory");
        return;
    }
    const int lane = threadIdx.x;
    double acc = 0.0, r = 1.0 + lane * 1e-6;
    long long t0 = clock64();
    if (V == 0) {
#pragma unroll 16
        for (int i = 0; i < N; ++i) acc = __dadd_rn(acc, r);
    } else if (V == 1 || V == 4 || V == 5) {
        for (int b = 0; b < N / U; ++b) {
            if (V == 5) asm volatile("bar.sync 1, 64;" ::: "memory");
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = sm[b * U + u + (lane & 1)];
#pragma unroll
            for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, v[u]);
            if (V == 4) __syncwarp();
        }
    } else if (V == 2) {
        const double2* s2 = reinterpret_cast<const double2*>(sm);
        for (int b = 0; b < N / U; ++b) {
            double2 v[U / 2];
#pragma unroll
            for (int u = 0; u < U / 2; ++u) v[u] = s2[b * U / 2 + u];
#pragma unroll
            for (int u = 0; u < U / 2; ++u) {
                acc = __dadd_rn(acc, v[u].x);
                acc = __dadd_rn(acc, v[u].y);
            }
        }
    } else if (V == 6 || V == 7) {
        // products formed one loop iteration ahead (loop-carried registers, so
        // ptxas cannot sink the DMULs next to their DADDs); V7 also carries
        // the operands one more iteration ahead
        double pr[U], xa[U], ya[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(sm[u], sm[u + 1 + (lane & 1)]);
        if (V == 7) {
#pragma unroll
            for (int u = 0; u < U; ++u) { xa[u] = sm[U + u]; ya[u] = sm[U + u + 1 + (lane & 1)]; }
        }
#pragma unroll 1
        for (int b = 0; b < N / U - 2; ++b) {
            double np[U];
            if (V == 6) {
#pragma unroll
                for (int u = 0; u < U; ++u) np[u] = __dmul_rn(sm[(b + 1) * U + u], sm[(b + 1) * U + u + 1 + (lane & 1)]);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) np[u] = __dmul_rn(xa[u], ya[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) { xa[u] = sm[(b + 2) * U + u]; ya[u] = sm[(b + 2) * U + u + 1 + (lane & 1)]; }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, pr[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) pr[u] = np[u];
        }
    } else if (V == 3) {
        for (int b = 0; b < N / U; ++b) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __dmul_rn(sm[b * U + u], sm[b * U + u + 1 + (lane & 1)]);
#pragma unroll
            for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, v[u]);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const char* names[] = {"register addend", "LDS batch of 16", "LDS.128 batch", "DMUL of LDS operands",
                           "LDS batch + syncwarp", "LDS batch, bar.sync with a 2nd warp",
                           "DMUL products one iteration ahead", "... + operands two iterations ahead"};
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 8; ++v) {
            long long h = 0;
            switch (v) {
            case 0: k<0><<<1, 32>>>(out, cyc); break;
            case 1: k<1><<<1, 32>>>(out, cyc); break;
            case 2: k<2><<<1, 32>>>(out, cyc); break;
            case 3: k<3><<<1, 32>>>(out, cyc); break;
            case 4: k<4><<<1, 32>>>(out, cyc); break;
            case 5: k<5><<<1, 64>>>(out, cyc); break;
            case 6: k<6><<<1, 32>>>(out, cyc); break;
            case 7: k<7><<<1, 32>>>(out, cyc); break;
            }
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-38s %.2f cycles/step\n", names[v], (double)h / N);
        }
    }
    return 0;
}
