// Chain-kernel gap probe (round 2): the column-major chain kernel of the
// session-2 experiment (88.5 us per phase at cfg 2 = 10.6 cycles/step) against
// the 8.6 cycles/step its inner loop reaches in isolation
// (chain_lds_probe.cu).  MODE 0: as in the library (TMA column segments);
// 1: the producer arrives on the full barriers without copying (no TMA
// traffic into shared memory); 2: as 1 and the consumers never wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o chain_gap_probe chain_gap_probe.cu
#include <cstdio>
#include "common.cuh"
using namespace coopcg_gpu;
constexpr int kChainWarps = 2;
constexpr int kChainU = 8, kChainLA = 2;
constexpr int kChainThreads = 32 * (1 + kChainWarps);
template <int T>
__host__ __device__ constexpr int chain_ts() { return T + 2; }
__host__ __device__ constexpr size_t chain_smem_bytes(int P, int T, int S, int nsrc) {
    return static_cast<size_t>(S) * nsrc * P * (T + 2) * sizeof(double) + 2 * S * sizeof(uint64_t);
}
template <int P, int T, int S, int MODE>
__global__ void __launch_bounds__(kChainThreads)
    gap_kernel(const double* __restrict__ s0, const double* __restrict__ s1,
                 const double* __restrict__ s2, int nsrc, int n, int ld,
                 int nchains, double* __restrict__ out, long long* cyc) {
    constexpr int U = kChainU, LA = kChainLA;
    constexpr int NBT = T / U;  // batches per tile
    constexpr int TS = chain_ts<T>();
    static_assert(U % 2 == 0, "operands come in LDS.128 pairs along k");
    static_assert(T % U == 0 && NBT % LA == 0, "register sets rotate within a tile");
    static_assert(LA + 1 < NBT, "loads run at most one tile ahead");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* cm = reinterpret_cast<double*>(smem_raw);  // [S][nsrc][P][TS]
    uint64_t* full = reinterpret_cast<uint64_t*>(cm + static_cast<size_t>(S) * nsrc * P * TS);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ntiles = (n + T - 1) / T;
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kChainWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        // producer: one lane copies the column segments of tile t into stage t % S
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                // an even number of rows (16-byte copies): a copied row past n is
                // the column's padding (cm_ld >= n rounded up to 16), never added
                const int rows = (min(T, n - t * T) + 1) & ~1;
                const uint32_t bytes = static_cast<uint32_t>(rows) * 8u;
                if (MODE == 1 || MODE == 2) {
                    mbar_arrive(&full[s]);
                } else {
                mbar_arrive_expect_tx(&full[s], bytes * P * nsrc);
                double* dst = cm + static_cast<size_t>(s) * nsrc * P * TS;
                for (int si = 0; si < nsrc; ++si) {
                    const double* src = (si == 0 ? s0 : (si == 1 ? s1 : s2)) + static_cast<size_t>(t) * T;
#pragma unroll 4
                    for (int c = 0; c < P; ++c)
                        bulk_g2s(dst + (si * P + c) * TS, src + static_cast<size_t>(c) * ld, bytes, &full[s]);
                }
                }
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int c = blockIdx.x * (kChainWarps * 32) + (tid - 32);
    const int dsx = 0, da = (c / P) % P, dsy = 1, db = c % P;  // the Gram phase: D_i . Q_j
    const int xoff = (dsx * P + da) * TS;
    const int yoff = (dsy * P + db) * TS;
    const int nb = (n + U - 1) / U;  // batches; all full except possibly the last
    auto tile_wait = [&](int t) {
        if (MODE != 2 && t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    // Operand batches (U steps) rotate through LA register sets, batch j in set
    // j % LA (the pipelined A.D's scheme): step q of a tile adds batch q's
    // products, forms batch q+1's from set (q+1) % LA and refills that set with
    // batch q+1+LA.  Loads run LA batches ahead of their DMUL, the DMUL one
    // batch ahead of its DADD, and every address is a per-tile stage pointer
    // plus a constant (q is a constant of the unrolled tile body).  Batches
    // past the last tile read stale ring data, multiplied, never added.
    double acc = 0.0;
    double pr[U], sx[LA][U], sy[LA][U];
    auto load_at = [&](const double* xb, const double* yb, double (&x)[U], double (&y)[U]) {
#pragma unroll
        for (int u = 0; u < U; u += 2) {
            const double2 xv = *reinterpret_cast<const double2*>(xb + u);
            const double2 yv = *reinterpret_cast<const double2*>(yb + u);
            x[u] = xv.x;
            x[u + 1] = xv.y;
            y[u] = yv.x;
            y[u + 1] = yv.y;
        }
    };
    auto load_q = [&](int qq, const double* x0, const double* y0, const double* x1, const double* y1,
                      double (&x)[U], double (&y)[U]) {
        if (qq < NBT) load_at(x0 + qq * U, y0 + qq * U, x, y);
        else load_at(x1 + (qq - NBT) * U, y1 + (qq - NBT) * U, x, y);
    };
    auto step = [&](int q, const double* x0, const double* y0, const double* x1, const double* y1) {
        const int sf = (q + 1) % LA;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc = __dadd_rn(acc, pr[u]);
            pr[u] = __dmul_rn(sx[sf][u], sy[sf][u]);
        }
        load_q(q + 1 + LA, x0, y0, x1, y1, sx[sf], sy[sf]);
    };
    auto stage = [&](int t) { return cm + static_cast<size_t>(t % S) * nsrc * P * TS; };
    const long long t_start = clock64();
    tile_wait(0);
    {
        const double *x0 = stage(0) + xoff, *y0 = stage(0) + yoff, *x1 = stage(1) + xoff, *y1 = stage(1) + yoff;
        double x[U], y[U];
        load_at(x0, y0, x, y);
#pragma unroll
        for (int u = 0; u < U; ++u) pr[u] = __dmul_rn(x[u], y[u]);
#pragma unroll
        for (int j = 1; j <= LA; ++j) load_q(j, x0, y0, x1, y1, sx[j % LA], sy[j % LA]);
    }
    // Tile t+1 is waited for just before the first step that loads from it
    // (the last LA + 1 steps of tile t), so the producer transposes it while
    // tile t is being summed: two column-major stages suffice.
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
        const double *x0 = stage(t) + xoff, *y0 = stage(t) + yoff;
        const double *x1 = stage(t + 1) + xoff, *y1 = stage(t + 1) + yoff;
        const int b0 = t * NBT;
        if ((t + 1) * T <= n) {
#pragma unroll
            for (int q = 0; q < NBT; ++q) {
                if (q == NBT - LA - 1) tile_wait(t + 1);
                step(q, x0, y0, x1, y1);
            }
        } else {
            // partial last tile: the batches that hold rows, the last one masked
#pragma unroll
            for (int q = 0; q < NBT; ++q) {
                // (no early exit: q stays a constant of the unrolled body, so
                // the register sets stay in registers)
                if (b0 + q < nb - 1) {
                    step(q, x0, y0, x1, y1);
                } else if (b0 + q == nb - 1) {
                    const int rem = n - (b0 + q) * U;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < rem) acc = __dadd_rn(acc, pr[u]);
                }
            }
        }
        __syncwarp();
        mbar_arrive_lane0(&empty[t % S], lane);
    }
    if (c < nchains) out[c] = acc;
    if (tid == 32) cyc[0] = clock64() - t_start;
}
template <int MODE>
void run(const char* name, const double* s0, const double* s1, const double* s2, int n, int ld, double* out,
         long long* cyc) {
    constexpr int P = 8, T = 256, S = 4;
    const size_t smem = chain_smem_bytes(P, T, S, 3);
    cudaFuncSetAttribute(gap_kernel<P, T, S, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h = 0;
    for (int r = 0; r < 3; ++r) {
        gap_kernel<P, T, S, MODE><<<1, kChainThreads, smem>>>(s0, s1, s2, 3, n, ld, 64, out, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-52s %6.2f cycles/step\n", name, (double)h / n);
}
int main() {
    const int n = 16384, P = 8, ld = n;
    double *s0, *s1, *s2, *out;
    long long* cyc;
    cudaMalloc(&s0, sizeof(double) * P * ld);
    cudaMalloc(&s1, sizeof(double) * P * ld);
    cudaMalloc(&s2, sizeof(double) * P * ld);
    {
        double* h = new double[(size_t)P * ld];
        for (size_t i = 0; i < (size_t)P * ld; ++i) h[i] = 1.0 + 1e-3 * (double)(i % 977);
        cudaMemcpy(s0, h, sizeof(double) * P * ld, cudaMemcpyHostToDevice);
        cudaMemcpy(s1, h, sizeof(double) * P * ld, cudaMemcpyHostToDevice);
        cudaMemcpy(s2, h, sizeof(double) * P * ld, cudaMemcpyHostToDevice);
        delete[] h;
    }
    cudaMalloc(&out, 1 << 16);
    cudaMalloc(&cyc, 8);
    run<0>("library chain kernel (TMA column segments)", s0, s1, s2, n, ld, out, cyc);
    run<1>("no copies (barrier arrivals only)", s0, s1, s2, n, ld, out, cyc);
    run<2>("no copies, consumers never wait", s0, s1, s2, n, ld, out, cyc);
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
