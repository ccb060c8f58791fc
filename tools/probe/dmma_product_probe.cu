// Can the FP64 tensor core form the exact mode's products?  One m8n8k4 DMMA
// with only k-slot 0 populated (A[:,0] = 8 row values, B[0,:] = 8 column
// values, the other slots zero, C = 0) gives the 8 x 8 outer product; each
// element is a*b + 0 + 0 + 0 + 0, i.e. RN(a*b) whatever the internal order --
// the DMUL result, up to the sign of a zero product (-0 vs +0), which a chain
// acc + p starting at +0 cannot see.  (1) exactness against __dmul_rn over
// random, tiny (subnormal-product), huge and special values; (2) throughput
// of a DADD-chain step mix: all products by DMUL vs a share by DMMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_product_probe dmma_product_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// A fragment: thread (g = lane/4, tg = lane%4) holds A[g][tg]; B fragment:
// B[tg][g]; C/D: thread holds D[g][2tg], D[g][2tg+1].
__global__ void exact_check(const double* __restrict__ av, const double* __restrict__ bv, int trials,
                            unsigned long long* mism, unsigned long long* zsign) {
    const int lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
    const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    for (int t = w; t < trials; t += gridDim.x * (blockDim.x / 32)) {
        const double* a8 = av + (size_t)t * 8;
        const double* b8 = bv + (size_t)t * 8;
        const double a = (tg == 0) ? a8[g] : 0.0;
        const double b = (tg == 0) ? b8[g] : 0.0;
        double c0 = 0.0, c1 = 0.0;
        dmma884(c0, c1, a, b);
        const double r0 = __dmul_rn(a8[g], b8[2 * tg]), r1 = __dmul_rn(a8[g], b8[2 * tg + 1]);
        auto cmp = [&](double x, double r) {
            if (x == r && std::signbit(x) == std::signbit(r)) return;
            if (x == 0.0 && r == 0.0) {
                atomicAdd(zsign, 1ull);  // +0 vs -0 only
                return;
            }
            if (x != x && r != r) return;  // both NaN
            atomicAdd(mism, 1ull);
        };
        cmp(c0, r0);
        cmp(c1, r1);
    }
}

// throughput: per k-step each thread adds 8 products into 8 chains (DADD);
// MODE 0: all 8 products by DMUL; MODE 1: 2 of 8 by one DMMA (2 products per
// thread), 6 by DMUL; MODE 2: 4 of 8 by two DMMAs.
template <int MODE>
__global__ void mix(const double* __restrict__ in, double* out, long long* cyc, int steps) {
    double acc[8], x[8], y[8];
    for (int i = 0; i < 8; ++i) {
        acc[i] = 0.0;
        x[i] = in[(threadIdx.x + i) & 63];
        y[i] = in[(threadIdx.x + 3 * i) & 63];
    }
    const long long t0 = clock64();
    for (int k = 0; k < steps; ++k) {
        double p[8];
        int first = 0;
        if (MODE >= 1) {
            double c0 = 0.0, c1 = 0.0;
            dmma884(c0, c1, x[0], y[0]);
            p[0] = c0;
            p[1] = c1;
            first = 2;
        }
        if (MODE >= 2) {
            double c0 = 0.0, c1 = 0.0;
            dmma884(c0, c1, x[1], y[1]);
            p[2] = c0;
            p[3] = c1;
            first = 4;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i >= first) p[i] = __dmul_rn(x[i], y[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __dadd_rn(acc[i], p[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(x[i], 1e-300);  // vary operands a little
    }
    const long long t1 = clock64();
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

static double rnd(uint64_t& s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(s >> 11) * 0x1.0p-53;
}

int main() {
    const int trials = 1 << 20;
    double* ha = new double[(size_t)trials * 8];
    double* hb = new double[(size_t)trials * 8];
    uint64_t s = 7;
    for (size_t i = 0; i < (size_t)trials * 8; ++i) {
        const int kind = (int)(rnd(s) * 10);
        double a = rnd(s) * 2 - 1, b = rnd(s) * 2 - 1;
        if (kind == 0) { a *= 1e-160; b *= 1e-160; }          // subnormal / zero products
        else if (kind == 1) { a *= 1e-300; }                   // tiny
        else if (kind == 2) { a *= 1e200; b *= 1e150; }        // overflow to inf
        else if (kind == 3) { a = -0.0; }
        else if (kind == 4) { a = std::ldexp(1.0 + rnd(s), -1022); b = 0.5 + rnd(s) * 1e-3; }  // near the subnormal edge
        else if (kind == 5) { a = 1.0 + rnd(s) * 0x1.0p-40; b = 1.0 - rnd(s) * 0x1.0p-40; }   // rounding ties region
        ha[i] = a;
        hb[i] = b;
    }
    double *da, *db;
    unsigned long long *mism, *zs;
    cudaMalloc(&da, sizeof(double) * trials * 8);
    cudaMalloc(&db, sizeof(double) * trials * 8);
    cudaMalloc(&mism, 8);
    cudaMalloc(&zs, 8);
    cudaMemcpy(da, ha, sizeof(double) * trials * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb, sizeof(double) * trials * 8, cudaMemcpyHostToDevice);
    cudaMemset(mism, 0, 8);
    cudaMemset(zs, 0, 8);
    exact_check<<<296, 256>>>(da, db, trials, mism, zs);
    unsigned long long hm = 0, hz = 0;
    cudaMemcpy(&hm, mism, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hz, zs, 8, cudaMemcpyDeviceToHost);
    printf("DMMA one-slot products vs DMUL over %d x 64 products: %llu mismatches, %llu +0/-0 sign-only differences\n",
           trials, hm, hz);
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    long long hc;
    const int steps = 4096;
    for (int warps : {1, 2, 4, 8}) {
        mix<0><<<1, 32 * warps>>>(da, out, cyc, steps);
        mix<0><<<1, 32 * warps>>>(da, out, cyc, steps);
        cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
        const double c0 = (double)hc / steps;
        mix<1><<<1, 32 * warps>>>(da, out, cyc, steps);
        mix<1><<<1, 32 * warps>>>(da, out, cyc, steps);
        cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
        const double c1 = (double)hc / steps;
        mix<2><<<1, 32 * warps>>>(da, out, cyc, steps);
        mix<2><<<1, 32 * warps>>>(da, out, cyc, steps);
        cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
        const double c2 = (double)hc / steps;
        printf("%d warps/SM: cycles per step (8 DADD + products; +8 DADD operand updates): "
               "all DMUL %.1f | 2 of 8 by DMMA %.1f | 4 of 8 by DMMA %.1f\n", warps, c0, c1, c2);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
