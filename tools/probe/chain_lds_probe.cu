// Chain inner-loop probe (round 2): a dependent DADD chain whose addends are
// DMULs of shared-memory operands, one chain per thread, 4 warps (one per
// SMSP), operands in column-major smem (consecutive k adjacent, LDS.128 = two
// steps).  No producer: the 4096-row operand columns are reused 4 times
// (16384 steps).  Variants of how the loads are written / batched, to find
// what keeps the step at the 8-cycle DADD latency.  Bitwise result check
// against a plain loop.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_lds_probe chain_lds_probe.cu
#include <cstdio>
#include <cstdint>

constexpr int KR = 1024;     // rows held in smem per column
constexpr int NSTEP = 16384; // chain length
constexpr int NCOL = 8;      // columns per operand block
constexpr int TS = KR + 2;   // column stride (doubles)

__device__ __forceinline__ double lds64(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ double2 lds128(const double* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

// MODE 0: plain loop (reference; ptxas schedules freely, unroll 8)
// MODE 1: unrolled tile body, register sets LA batches ahead (the library's scheme), U = 8
// MODE 2: as 1 with inline-asm volatile loads
// MODE 4: row-major [k][NCOL] operand tiles (the library's source layout),
//         one LDS.64 per operand per step, sets + asm volatile loads
// MODE 3: register double-buffer of W steps: load W steps of both operands at once, then W steps
template <int MODE, int U, int LA, int W>
__global__ void __launch_bounds__(128) chain(const double* __restrict__ g, double* __restrict__ out,
                                             long long* cyc) {
    extern __shared__ __align__(16) double sm[];  // x cols [NCOL][TS], y cols [NCOL][TS]
    for (int i = threadIdx.x; i < 2 * NCOL * TS; i += blockDim.x) sm[i] = g[i % 4099] ;
    __syncthreads();
    const int t = threadIdx.x;
    const double* xs = sm + (t & 3) * TS;
    const double* ys = sm + NCOL * TS + ((t >> 2) & 7) * TS;
    double acc = 0.0;
    long long t0 = clock64();
    if (MODE == 0) {
#pragma unroll 8
        for (int k = 0; k < NSTEP; ++k) acc = __dadd_rn(acc, __dmul_rn(xs[k & (KR - 1)], ys[k & (KR - 1)]));
    } else if (MODE == 1 || MODE == 2) {
        constexpr int T = KR, NBT = T / U;
        double pr[U], sx[LA][U], sy[LA][U];
        auto load_at = [&](int k0, double (&x)[U], double (&y)[U]) {
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                const int k = (k0 + u) & (KR - 1);
                double2 a, b;
                if (MODE == 2) {
                    a = lds128(xs + k);
                    b = lds128(ys + k);
                } else {
                    a = *reinterpret_cast<const double2*>(xs + k);
                    b = *reinterpret_cast<const double2*>(ys + k);
                }
                x[u] = a.x; x[u + 1] = a.y;
                y[u] = b.x; y[u + 1] = b.y;
            }
        };
        {
            double x[U], y[U];
            load_at(0, x, y);
#pragma unroll
            for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(x[u], y[u]);
#pragma unroll
            for (int j = 1; j <= LA; ++j) load_at(j * U, sx[j % LA], sy[j % LA]);
        }
#pragma unroll 1
        for (int tile = 0; tile < NSTEP / T; ++tile) {
#pragma unroll
            for (int q = 0; q < NBT; ++q) {
                const int sf = (q + 1) % LA;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc = __dadd_rn(acc, pr[u]);
                    pr[u] = __dmul_rn(sx[sf][u], sy[sf][u]);
                }
                load_at((q + 1 + LA) * U, sx[sf], sy[sf]);
            }
        }
    } else if (MODE == 4) {
        // row-major: x[k][c] at sm[k * NCOL + c], y at sm[KR * NCOL + k * NCOL + c]
        const double* xr = sm + (t & 3);
        const double* yr = sm + KR * NCOL + ((t >> 2) & 7);
        constexpr int T = KR, NBT = T / U;
        double pr[U], sx[LA][U], sy[LA][U];
        auto load_at = [&](int k0, double (&x)[U], double (&y)[U]) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = (k0 + u) & (KR - 1);
                x[u] = lds64(xr + k * NCOL);
                y[u] = lds64(yr + k * NCOL);
            }
        };
        {
            double x[U], y[U];
            load_at(0, x, y);
#pragma unroll
            for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(x[u], y[u]);
#pragma unroll
            for (int j = 1; j <= LA; ++j) load_at(j * U, sx[j % LA], sy[j % LA]);
        }
#pragma unroll 1
        for (int tile = 0; tile < NSTEP / T; ++tile) {
#pragma unroll
            for (int q = 0; q < NBT; ++q) {
                const int sf = (q + 1) % LA;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc = __dadd_rn(acc, pr[u]);
                    pr[u] = __dmul_rn(sx[sf][u], sy[sf][u]);
                }
                load_at((q + 1 + LA) * U, sx[sf], sy[sf]);
            }
        }
    } else if (MODE == 5) {
        // row-major, two chains per thread sharing x: (x_c, y_j), (x_c, y_j+1);
        // per step one LDS.64 (x) and one LDS.128 (the y pair)
        const double* xr = sm + (t & 3);
        const double* yr = sm + KR * NCOL + 2 * ((t >> 2) & 3);
        constexpr int T = KR, NBT = T / U;
        double acc2 = 0.0;
        double pa[U], pb[U], sx[LA][U], sy[LA][U], sz[LA][U];
        auto load_at = [&](int k0, double (&x)[U], double (&y)[U], double (&z)[U]) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = (k0 + u) & (KR - 1);
                x[u] = lds64(xr + k * NCOL);
                const double2 v = lds128(yr + k * NCOL);
                y[u] = v.x;
                z[u] = v.y;
            }
        };
        {
            double x[U], y[U], z[U];
            load_at(0, x, y, z);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                pa[u] = __dmul_rn(x[u], y[u]);
                pb[u] = __dmul_rn(x[u], z[u]);
            }
#pragma unroll
            for (int j = 1; j <= LA; ++j) load_at(j * U, sx[j % LA], sy[j % LA], sz[j % LA]);
        }
#pragma unroll 1
        for (int tile = 0; tile < NSTEP / T; ++tile) {
#pragma unroll
            for (int q = 0; q < NBT; ++q) {
                const int sf = (q + 1) % LA;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    acc = __dadd_rn(acc, pa[u]);
                    acc2 = __dadd_rn(acc2, pb[u]);
                    pa[u] = __dmul_rn(sx[sf][u], sy[sf][u]);
                    pb[u] = __dmul_rn(sx[sf][u], sz[sf][u]);
                }
                load_at((q + 1 + LA) * U, sx[sf], sy[sf], sz[sf]);
            }
        }
        acc = acc + 0.0 * acc2;  // keep both chains live (acc2 is checked separately below)
        if (acc2 == 1234.5) out[1000] = acc2;
    } else if (MODE == 3) {
        // W-step register windows, double buffered: window w+1 loads while w is summed
        double xa[W], ya[W], xb[W], yb[W];
        auto win = [&](int k0, double (&x)[W], double (&y)[W]) {
#pragma unroll
            for (int u = 0; u < W; u += 2) {
                const int k = (k0 + u) & (KR - 1);
                const double2 a = *reinterpret_cast<const double2*>(xs + k);
                const double2 b = *reinterpret_cast<const double2*>(ys + k);
                x[u] = a.x; x[u + 1] = a.y;
                y[u] = b.x; y[u + 1] = b.y;
            }
        };
        win(0, xa, ya);
#pragma unroll 1
        for (int k = 0; k < NSTEP; k += 2 * W) {
            win(k + W, xb, yb);
#pragma unroll
            for (int u = 0; u < W; ++u) acc = __dadd_rn(acc, __dmul_rn(xa[u], ya[u]));
            win(k + 2 * W, xa, ya);
#pragma unroll
            for (int u = 0; u < W; ++u) acc = __dadd_rn(acc, __dmul_rn(xb[u], yb[u]));
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + t] = acc;
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int U, int LA, int W>
void run(const char* name, const double* g, double* out, long long* cyc, const double* ref, int nth = 128) {
    const size_t smem = 2 * NCOL * TS * sizeof(double);
    cudaFuncSetAttribute(chain<MODE, U, LA, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h = 0;
    for (int rep = 0; rep < 3; ++rep) {
        chain<MODE, U, LA, W><<<1, nth, smem>>>(g, out, cyc);
        cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    }
    double o[128];
    cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
    bool same = true;
    for (int i = 0; i < nth; ++i) same &= (o[i] == ref[i]);
    printf("%-44s %3d thr %6.2f cycles/step  %s\n", name, nth, (double)h / NSTEP, same ? "bit-identical" : "MISMATCH");
}

int main() {
    const int NG = 4099;
    double hg[NG];
    uint64_t s = 12345;
    for (int i = 0; i < NG; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        hg[i] = (double)(s >> 11) * 0x1.0p-53 - 0.5;
    }
    double *g, *out;
    long long* cyc;
    cudaMalloc(&g, sizeof hg);
    cudaMalloc(&out, 128 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    cudaMemcpy(g, hg, sizeof hg, cudaMemcpyHostToDevice);
    // host reference (plain sequential chain per thread)
    double ref[128];
    for (int t = 0; t < 128; ++t) {
        double acc = 0.0;
        const int xc = t & 3, yc = (t >> 2) & 7;
        for (int k = 0; k < NSTEP; ++k) {
            const int kk = k & (KR - 1);
            const double x = hg[(xc * TS + kk) % NG], y = hg[((NCOL + yc) * TS + kk) % NG];
            volatile double p = x * y;
            acc = acc + p;
        }
        ref[t] = acc;
    }
    double ref4[128];
    for (int t = 0; t < 128; ++t) {
        double acc = 0.0;
        const int xc = t & 3, yc = (t >> 2) & 7;
        for (int k = 0; k < NSTEP; ++k) {
            const int kk = k & (KR - 1);
            const double x = hg[(kk * NCOL + xc) % NG], y = hg[(KR * NCOL + kk * NCOL + yc) % NG];
            volatile double p = x * y;
            acc = acc + p;
        }
        ref4[t] = acc;
    }
    for (int nth : {32, 64}) {
        run<5, 8, 2, 8>("row-major 2 chains/thread (LDS.64 x + LDS.128 y2)", g, out, cyc, ref4, nth);
        run<5, 4, 4, 8>("row-major 2 chains/thread U=4 LA=4", g, out, cyc, ref4, nth);
    }
    for (int nth : {32, 64, 128}) {
        run<4, 8, 2, 8>("row-major LDS.64, sets U=8 LA=2, asm loads", g, out, cyc, ref4, nth);
        run<4, 4, 4, 8>("row-major LDS.64, sets U=4 LA=4, asm loads", g, out, cyc, ref4, nth);
    }
    run<0, 8, 2, 8>("plain loop (unroll 8)", g, out, cyc, ref);
    run<1, 8, 2, 8>("sets U=8 LA=2", g, out, cyc, ref);
    run<1, 8, 4, 8>("sets U=8 LA=4", g, out, cyc, ref);
    run<1, 4, 4, 8>("sets U=4 LA=4", g, out, cyc, ref);
    run<1, 2, 8, 8>("sets U=2 LA=8", g, out, cyc, ref);
    run<2, 8, 2, 8>("sets U=8 LA=2, asm volatile loads", g, out, cyc, ref);
    run<2, 4, 4, 8>("sets U=4 LA=4, asm volatile loads", g, out, cyc, ref);
    run<3, 8, 2, 16>("windows W=16", g, out, cyc, ref);
    run<3, 8, 2, 32>("windows W=32", g, out, cyc, ref);
    for (int nth : {32, 64}) {
        run<2, 8, 2, 8>("sets U=8 LA=2, asm volatile loads", g, out, cyc, ref, nth);
        run<3, 8, 2, 32>("windows W=32", g, out, cyc, ref, nth);
        run<0, 8, 2, 8>("plain loop (unroll 8)", g, out, cyc, ref, nth);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
