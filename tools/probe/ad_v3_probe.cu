// A.D (exact) redesign probe: thread = RPT rows x CPT columns, operands
// software-pipelined two batches ahead in two register sets (the chain
// kernel's scheme), one straight-line loop body per tile.  Goal: fewer
// shared-memory wavefronts per MAC than ad_exact_kernel (6 per 128 MACs there;
// 8 per 256 MACs at RPT=2, CPT=4) without losing the latency hiding.
// Sweeps shapes at n=16384, P=8 and checks sampled rows bitwise against a
// sequential CPU restatement (k ascending, separate roundings).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1204_0069_b200/csrc -o ad_v3_probe ad_v3_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "exact_kernels.cuh"

using namespace coopcg_gpu;

template <int P, int CPT, int RPT, int BR, int T, int S, int U, int DL = 2>
__global__ void __launch_bounds__(32 + 32 * ((BR / RPT * (P / CPT) + 31) / 32))
    ad_v3(const double* __restrict__ Ap, int n, const double* __restrict__ D, double* __restrict__ Y) {
    constexpr int RG = BR / RPT;
    constexpr int NT = RG * (P / CPT);
    constexpr int NW = (NT + 31) / 32;
    constexpr int NBT = T / U;
    static_assert(T % (2 * U) == 0, "even batches per tile");
    static_assert(RPT == 1 || RPT == 2, "rows per thread");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Ds = As + S * T * BR;
    uint64_t* full = reinterpret_cast<uint64_t*>(Ds + S * T * P);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (n + T - 1) / T;
    const double* panel = Ap + static_cast<size_t>(blockIdx.x) * n * BR;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int k0 = t * T;
                const int rows = min(T, n - k0);
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows) * (BR * 8u + P * 8u));
                bulk_g2s_evict_first(As + s * T * BR, panel + static_cast<size_t>(k0) * BR,
                                     static_cast<uint32_t>(rows) * BR * 8u, &full[s], pol);
                bulk_g2s(Ds + s * T * P, D + static_cast<size_t>(k0) * P, static_cast<uint32_t>(rows) * P * 8u,
                         &full[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int tid = threadIdx.x - 32;
    const int rr = tid % RG;
    const int g = min(tid / RG, P / CPT - 1);
    const int aoff = rr * RPT;
    const int doff = g * CPT;
    auto tile_wait = [&](int t) {
        if (t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    // k-step kk of batch j: stage (j / NBT) % S, row (j % NBT) * U + u
    auto abase = [&](int j) -> const double* {
        return As + ((j / NBT) % S) * T * BR + (j % NBT) * U * BR + aoff;
    };
    auto dbase = [&](int j) -> const double* {
        return Ds + ((j / NBT) % S) * T * P + (j % NBT) * U * P + doff;
    };
    double acc[RPT][CPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[r][c] = 0.0;
    double pr[U][RPT][CPT];
    double ae[U][RPT], ao[U][RPT], de[U][CPT], dq[U][CPT];
    auto load = [&](int j, double (&a)[U][RPT], double (&d)[U][CPT]) {
        const double* ab = abase(j);
        const double* db = dbase(j);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (RPT == 2) {
                const double2 v = *reinterpret_cast<const double2*>(ab + u * BR);
                a[u][0] = v.x;
                a[u][RPT - 1] = v.y;
            } else {
                a[u][0] = ab[u * BR];
            }
            if (DL == 2) {
#pragma unroll
                for (int c = 0; c < CPT / 2; ++c) {
                    const double2 v = reinterpret_cast<const double2*>(db + u * P)[c];
                    d[u][2 * c] = v.x;
                    d[u][2 * c + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int c = 0; c < CPT; ++c) d[u][c] = db[u * P + c];
            }
        }
    };
    // add batch b, form batch b+1 (from a/d r-set), load batch b+2 (w-set)
    auto step = [&](int b, const double (&ar)[U][RPT], const double (&dr)[U][CPT], double (&aw)[U][RPT],
                    double (&dw)[U][CPT]) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
                    acc[r][c] = __dadd_rn(acc[r][c], pr[u][r][c]);
                    pr[u][r][c] = __dmul_rn(ar[u][r], dr[u][c]);
                }
        load(b + 2, aw, dw);
    };
    tile_wait(0);
    {
        double a0[U][RPT], d0[U][CPT];
        load(0, a0, d0);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int c = 0; c < CPT; ++c) pr[u][r][c] = __dmul_rn(a0[u][r], d0[u][c]);
        load(1, ao, dq);
    }
    const int nb = (n + U - 1) / U;
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
        tile_wait(t + 1);
        const int b0 = t * NBT;
        if ((t + 1) * T <= n) {
#pragma unroll
            for (int q = 0; q < NBT; q += 2) {
                step(b0 + q, ao, dq, ae, de);
                step(b0 + q + 1, ae, de, ao, dq);
            }
        } else {
            for (int q = 0; q < NBT && b0 + q < nb; ++q) {
                const int b = b0 + q;
                if (b == nb - 1) {
                    const int rem = n - b * U;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < rem)
#pragma unroll
                            for (int r = 0; r < RPT; ++r)
#pragma unroll
                                for (int c = 0; c < CPT; ++c) acc[r][c] = __dadd_rn(acc[r][c], pr[u][r][c]);
                } else if (q & 1) {
                    step(b, ae, de, ao, dq);
                } else {
                    step(b, ao, dq, ae, de);
                }
            }
        }
        __syncwarp();
        mbar_arrive_lane0(&empty[t % S], lane);
    }
    if (tid < NT) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int row = blockIdx.x * BR + aoff + r;
            if (row < n)
#pragma unroll
                for (int c = 0; c < CPT; ++c) Y[static_cast<size_t>(row) * P + doff + c] = acc[r][c];
        }
    }
}

__host__ __device__ inline double aval(int i, int k) {
    unsigned h = (unsigned)i * 2654435761u ^ ((unsigned)k * 40503u + 0x9e3779b9u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    return ((h & 0xffffff) / 16777216.0 - 0.5) * 1.37;
}
__host__ __device__ inline double dval(int k, int c) { return aval(k + 7919, c * 31 + 3) * 3.1; }

__global__ void fill_panels(double* Ap, int n, int BR) {
    const size_t tot = (size_t)((n + BR - 1) / BR) * BR * n;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const size_t pn = e / ((size_t)n * BR);
        const size_t rem = e % ((size_t)n * BR);
        const int k = (int)(rem / BR), r = (int)(rem % BR);
        const int i = (int)(pn * BR + r);
        Ap[e] = (i < n) ? aval(i, k) : 0.0;
    }
}
__global__ void fill_d(double* D, int n, int P) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * P; e += gridDim.x * blockDim.x) D[e] = dval(e / P, e % P);
}

static double* g_Ap;
static double *g_D, *g_Y;
static std::vector<double> g_ref;  // sampled rows x P
static std::vector<int> g_rows;

template <int P, int CPT, int RPT, int BR, int T, int S, int U, int DL = 2>
void run(int n, const char* tag) {
    auto k = ad_v3<P, CPT, RPT, BR, T, S, U, DL>;
    const size_t smem = (size_t)S * T * (BR + P) * 8 + 2 * S * 8;
    if (smem > 227 * 1024) {
        std::printf("%s: smem %zu too big\n", tag, smem);
        return;
    }
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0;
    constexpr int NW0 = ((BR / RPT) * (P / CPT) + 31) / 32;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 + 32 * NW0, smem);
    fill_panels<<<148 * 8, 256>>>(g_Ap, n, BR);
    cudaMemset(g_Y, 0xff, (size_t)n * P * 8);
    constexpr int NW = ((BR / RPT) * (P / CPT) + 31) / 32;
    dim3 grid((n + BR - 1) / BR), block(32 + 32 * NW);
    k<<<grid, block, smem>>>(g_Ap, n, g_D, g_Y);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> y((size_t)n * P);
    cudaMemcpy(y.data(), g_Y, y.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (size_t q = 0; q < g_rows.size(); ++q)
        for (int c = 0; c < P; ++c)
            if (y[(size_t)g_rows[q] * P + c] != g_ref[q * P + c]) ++bad;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k<<<grid, block, smem>>>(g_Ap, n, g_D, g_Y);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    std::printf("%-30s P=%d CPT=%d RPT=%d BR=%3d T=%3d S=%d U=%d DL=%d grid=%4d warps=%d occ=%d smem=%6zu : %8.1f us  "
                "%5.2f TF/s  bad=%d %s\n",
                tag, P, CPT, RPT, BR, T, S, U, DL, grid.x, NW, occ, smem, ms * 1e3, 2.0 * n * n * P / (ms * 1e-3) / 1e12, bad,
                e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int P, int CPT, int BR, int T, int S, int RPT = 1>
void run_cur(int n) {  // the production kernel (same layout fill)
    auto k = (RPT == 1) ? ad_exact_kernel<P, CPT, BR, T, S> : ad_exact_rpt_kernel<P, CPT, BR, T, S, 2>;
    const size_t smem = (size_t)S * T * (BR + P) * 8 + 2 * S * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fill_panels<<<148 * 8, 256>>>(g_Ap, n, BR);
    dim3 grid((n + BR - 1) / BR), block(32 + 32 * ad_consumer_warps(BR / RPT, P / CPT));
    k<<<grid, block, smem>>>(g_Ap, n, n, 0, g_D, g_Y, nullptr, P, nullptr, PeerRows{});
    cudaDeviceSynchronize();
    std::vector<double> y((size_t)n * P);
    cudaMemcpy(y.data(), g_Y, y.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (size_t q = 0; q < g_rows.size(); ++q)
        for (int c = 0; c < P; ++c)
            if (y[(size_t)g_rows[q] * P + c] != g_ref[q * P + c]) ++bad;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k<<<grid, block, smem>>>(g_Ap, n, n, 0, g_D, g_Y, nullptr, P, nullptr, PeerRows{});
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    std::printf("%-30s P=%d CPT=%d RPT=%d BR=%3d T=%3d S=%d : %8.1f us  bad=%d\n", "current ad_exact", P, CPT, RPT, BR,
                T, S, ms * 1e3, bad);
}

template <int P>
void setup(int n) {
    g_rows.clear();
    g_ref.clear();
    fill_d<<<148 * 4, 256>>>(g_D, n, P);
    for (int q = 0; q < 48; ++q) g_rows.push_back((int)((q * 2654435761ull) % n));
    g_rows.push_back(n - 1);
    g_rows.push_back(0);
    for (int i : g_rows)
        for (int c = 0; c < P; ++c) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) {
                volatile double prod = aval(i, k) * dval(k, c);
                acc = acc + prod;
            }
            g_ref.push_back(acc);
        }
}

int main(int argc, char** argv) {
    const char mode = argc > 1 ? argv[1][0] : '8';
    const size_t nmax = mode == '3' ? 131072 : mode == '1' ? 65536 : 16384;
    cudaMalloc(&g_Ap, (nmax + 256) * nmax * 8);
    cudaMalloc(&g_D, nmax * 32 * 8);
    cudaMalloc(&g_Y, nmax * 32 * 8);
    if (mode == '8') {
        const int n = 16384;
        setup<8>(n);
        run_cur<8, 4, 64, 64, 2>(n);
        run<8, 4, 2, 128, 64, 3, 2>(n, "rpt2 cpt4 4w");
        run<8, 4, 2, 128, 64, 3, 2, 1>(n, "rpt2 cpt4 4w D lds64");
        run<8, 4, 2, 64, 64, 3, 2>(n, "rpt2 cpt4 2w (2 cta/sm?)");
        run<8, 4, 2, 64, 48, 3, 2>(n, "rpt2 cpt4 2w T48");
        run<8, 4, 2, 128, 32, 6, 2>(n, "rpt2 cpt4 4w T32 S6");
        run<8, 4, 2, 128, 64, 3, 4>(n, "rpt2 cpt4 4w U4");
        run<8, 8, 2, 128, 64, 3, 2>(n, "rpt2 cpt8 2w");
        run<8, 2, 2, 64, 64, 3, 2>(n, "rpt2 cpt2 4w");
    } else if (mode == '1') {
        const int n = 65536;
        setup<16>(n);
        run_cur<16, 4, 64, 64, 2, 2>(n);
        run<16, 4, 2, 128, 64, 3, 2>(n, "p16 rpt2 cpt4 8w");
        run<16, 4, 2, 64, 64, 3, 2>(n, "p16 rpt2 cpt4 4w");
        run<16, 4, 2, 112, 64, 3, 2>(n, "p16 rpt2 cpt4 7w");
        run<16, 8, 2, 128, 64, 3, 2>(n, "p16 rpt2 cpt8 4w");
    } else if (mode == '4') {
        for (int n : {4096, 1000}) {
            setup<4>(n);
            run_cur<4, 2, 32, 256, 3>(n);
            run<4, 2, 1, 32, 128, 4, 2>(n, "p4 rpt1 cpt2 T128 S4 U2");
            run<4, 2, 1, 32, 128, 4, 4>(n, "p4 rpt1 cpt2 T128 S4 U4");
            run<4, 2, 1, 32, 128, 4, 8>(n, "p4 rpt1 cpt2 T128 S4 U8");
            run<4, 2, 1, 16, 128, 4, 4>(n, "p4 rpt1 cpt2 BR16 T128 S4 U4");
            run<4, 2, 1, 16, 128, 4, 8>(n, "p4 rpt1 cpt2 BR16 T128 S4 U8");
            run<4, 4, 1, 32, 128, 4, 4>(n, "p4 rpt1 cpt4 1w T128 S4 U4");
            run<4, 2, 1, 32, 64, 6, 4>(n, "p4 rpt1 cpt2 T64 S6 U4");
        }
    } else if (mode == 'c') {  // P = 8 at cfg-1-like small n: shapes for n <= 9472
        for (int n : {4096, 9472}) {
            setup<8>(n);
            run_cur<8, 4, 32, 64, 2>(n);
            run_cur<8, 4, 64, 64, 2>(n);
            run<8, 4, 2, 64, 64, 3, 2>(n, "p8 rpt2 cpt4 BR64");
            run<8, 4, 1, 32, 128, 4, 4>(n, "p8 rpt1 cpt4 BR32 T128 U4");
            run<8, 2, 1, 32, 128, 4, 4>(n, "p8 rpt1 cpt2 BR32 T128 U4");
            run<8, 4, 2, 128, 64, 3, 2>(n, "p8 rpt2 cpt4 BR128");
        }
    } else {
        const int n = 131072;
        setup<32>(n);
        run_cur<32, 4, 64, 64, 2, 2>(n);
        run<32, 4, 2, 64, 64, 3, 2>(n, "p32 rpt2 cpt4 8w");
        run<32, 4, 2, 32, 64, 3, 2>(n, "p32 rpt2 cpt4 4w");
        run<32, 8, 2, 64, 64, 3, 2>(n, "p32 rpt2 cpt8 4w");
    }
    return 0;
}
