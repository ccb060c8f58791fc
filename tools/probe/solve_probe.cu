// Phase timing (clock64) of the one-warp alpha solve at P = 8: where do the
// ~16k active cycles go?  Same code path as exact_kernels.cuh's
// alpha_solve_warp<8> (run by warp 0 of alpha_update_kernel), with timestamps between the phases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o solve_probe solve_probe.cu
#include <cstdio>
#include <vector>
#include "exact_kernels.cuh"
using namespace coopcg_gpu;

template <int P>
__global__ void __launch_bounds__(32) alpha_timed(double* __restrict__ small, Ctl* ctl, long long* ts) {
    long long t0 = clock64();
    if (*reinterpret_cast<volatile int*>(&ctl->stop)) return;
    __shared__ double lu[P][P + 1];
    __shared__ double rh[P][P + 1];
    __shared__ int perm[P];
    const int lane = threadIdx.x;
    const int p = ctl->p;
    long long t1 = clock64();
    const SmallLayout L{P};
    const double* raw = small + L.raw();
    double m[P];
    double maxabs = 0.0, diag = 0.0, nsq = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) m[j] = 0.0;
    if (lane < p) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            if (j < p) {
                m[j] = __dmul_rn(__dadd_rn(raw[lane * P + j], raw[j * P + lane]), 0.5);
                const double a = fabs(m[j]);
                maxabs = (maxabs < a) ? a : maxabs;
                if (j == lane) diag = m[j];
            }
            rh[lane][j] = small[L.rhs_a() + lane * P + j];
        }
        nsq = small[L.nsq_d() + lane];
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, maxabs, off);
        maxabs = (maxabs < o) ? o : maxabs;
    }
    const double floor = __dmul_rn(maxabs, 1e-14);
    const bool bad = (lane < p) && !(diag > 0.0) && (nsq > 0.0);
    if (__any_sync(0xffffffffu, bad)) return;
    long long t2 = clock64();
    int pv;
    if (!lu_factor_regs<P>(m, pv, lane, p, floor)) return;
    long long t3 = clock64();
    if (lane < P) {
#pragma unroll
        for (int j = 0; j < P; ++j) lu[lane][j] = m[j];
        perm[lane] = pv;
    }
    __syncwarp();
    long long t4 = 0, t5 = 0;
    if (lane < p) {
        double x[P];
        lu_solve_regs<P>(lu, perm, p, rh[lane], x);
        t4 = clock64();
#pragma unroll
        for (int j = 0; j < P; ++j) small[L.alpha() + lane * P + j] = (j < p) ? x[j] : 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j)
            if (j < p) ctl->lu[lane * p + j] = m[j];
        ctl->perm[lane] = pv;
        t5 = clock64();
    }
    if (lane == 0) {
        ts[0] = t1 - t0;
        ts[1] = t2 - t1;
        ts[2] = t3 - t2;
        ts[3] = t4 - t3;
        ts[4] = t5 - t4;
    }
}

int main() {
    const int P = 8, p = 8;
    SmallLayout L{P};
    std::vector<double> h(L.total(), 0.0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) {
            h[L.raw() + i * P + j] = (i == j ? 10.0 : 0.1 * (i + j)) + 0.01 * i;
            h[L.rhs_a() + i * P + j] = 1.0 + i - j;
        }
    for (int i = 0; i < p; ++i) h[L.nsq_d() + i] = 1.0;
    double* small;
    Ctl* ctl;
    long long* ts;
    cudaMalloc(&small, h.size() * 8);
    cudaMalloc(&ctl, sizeof(Ctl));
    cudaMalloc(&ts, 64);
    cudaMemcpy(small, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    Ctl hc{};
    hc.p = p;
    hc.P = P;
    cudaMemcpy(ctl, &hc, sizeof(Ctl), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
        alpha_timed<8><<<1, 32>>>(small, ctl, ts);
        long long t[5];
        cudaMemcpy(t, ts, sizeof(t), cudaMemcpyDeviceToHost);
        std::printf("stop+p %lld | loads+sym %lld | LU %lld | solve %lld | stores %lld cycles  (%s)\n", t[0], t[1], t[2],
                    t[3], t[4], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
