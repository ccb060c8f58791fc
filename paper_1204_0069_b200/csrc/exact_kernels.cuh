// exact_kernels.cuh -- bit-exact cCG iteration kernels for sm_100a.
//
// "Exact" = every output scalar is produced by the same sequence of IEEE
// double operations as the reference CPU solver (coopcg/kernels.hpp:13-16:
// ascending-index accumulation from +0.0, one rounding per multiply and per
// add -- the reference forbids FMA contraction, CMakeLists.txt:25).  Only
// the assignment of independent chains to threads differs.  Every multiply /
// add below is an explicit __dmul_rn / __dadd_rn so ptxas cannot contract.
#pragma once
#include "common.cuh"

namespace coopcg_gpu {

// ---------------------------------------------------------------------------
// (1) Q = A . D, the hot kernel.
//
// Reference: kernels::matvec_col (kernels.hpp:28-34) per column via
// stage_matvec (block_cg.hpp:146-151): Q[i][j] = sum_k A[i][k] * D[k][j], k
// ascending.  The reference streams A p times per iteration (once per
// agent); here A is streamed ONCE for all p columns.
//
// Device layout: A is stored in panels of BR rows (common.cuh ap_idx): a
// panel holds A(i, k) for its BR rows at k*BR + r, so the k-th step of 32
// consecutive row chains reads 256 contiguous bytes and a T x BR stage tile
// is ONE contiguous block.  A CTA owns one panel and all P columns split
// into P/CPT groups of CPT columns per thread; its A tiles and D tiles
// (T x P) stream through an S-stage shared-memory ring filled by bulk async
// copies (cp.async.bulk, TMA 1-D: one copy for A, one for D per stage)
// completing on mbarriers.  Each thread runs CPT independent sequential chains.
//
// Epilogue (sub_b != 0): Y = acc - b (block_cg.hpp:132-138 / :236-241
// `r[row] -= b[row]`), used for R0 = A X0 - b, the periodic residual
// recomputation and the final true residual (solvers.hpp:188-210).
// Consumer threads: BR rows x P/CPT column groups, rounded up to whole warps
// (BR need not be a power of two: the panel height is chosen to balance rows
// over the SMs, coopcg_gpu.cu pick_ad_config); surplus threads idle.
__host__ __device__ constexpr int ad_consumer_warps(int rows, int groups) { return (rows * groups + 31) / 32; }

// PUSH (peer mode only): store the rows into every rank's copy of Y through
// `peers` (a separate instantiation keeps the common path's code unchanged).
template <int P, int CPT, int BR, int T, int S, bool PUSH = false>
__global__ void __launch_bounds__(32 + 32 * ad_consumer_warps(BR, P / CPT))
    ad_exact_kernel(const double* __restrict__ Ap, int n, int n_loc, int row0,
                    const double* __restrict__ D, double* __restrict__ Y,
                    const double* __restrict__ b, int p, const int* __restrict__ stop, PeerRows peers,
                    int res_k) {
    pdl_wait();
    constexpr int kConsumerWarps = ad_consumer_warps(BR, P / CPT);
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Ds = As + S * T * BR;
    uint64_t* full = reinterpret_cast<uint64_t*>(Ds + S * T * P);
    uint64_t* empty = full + S;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.x * BR;
    const int ntiles = (n + T - 1) / T;
    const double* panel = Ap + static_cast<size_t>(blockIdx.x) * n * BR;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // Producer: one lane streams the A panel tiles and the D tiles.
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy(), pol_res = l2_evict_last_policy();
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int k0 = t * T;
                const int rows = min(T, n - k0);
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows) * (BR * 8u + P * 8u));
                bulk_g2s_evict_first(As + s * T * BR, panel + static_cast<size_t>(k0) * BR,
                                     static_cast<uint32_t>(rows) * BR * 8u, &full[s], k0 < res_k ? pol_res : pol);
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
    const int r = tid % BR;
    const int g = tid / BR;  // == P / CPT for the surplus threads (no output)
    const int gl = min(g, P / CPT - 1);
    double acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.0;

    int s = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&full[s], phase);
        const double* a_t = As + s * T * BR + r;
        const double* d_t = Ds + s * T * P + gl * CPT;
        const int rows = min(T, n - t * T);
        if (rows == T) {
            // Register software pipeline: the products of a batch of U k-steps
            // are formed, the next batch's shared-memory loads are issued, and
            // only then the dependent DADD chains run (k ascending per column).
            constexpr int U = (CPT >= 8) ? 2 : 4;
            static_assert(T % U == 0, "T must be a multiple of U");
            double av[U];
            double2 dv[U][CPT / 2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                av[u] = a_t[u * BR];
#pragma unroll
                for (int c = 0; c < CPT / 2; ++c) dv[u][c] = reinterpret_cast<const double2*>(d_t + u * P)[c];
            }
#pragma unroll
            for (int kb = 0; kb < T; kb += U) {
                double prod[U][CPT];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int c = 0; c < CPT / 2; ++c) {
                        prod[u][2 * c] = __dmul_rn(av[u], dv[u][c].x);
                        prod[u][2 * c + 1] = __dmul_rn(av[u], dv[u][c].y);
                    }
                if (kb + U < T) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        av[u] = a_t[(kb + U + u) * BR];
#pragma unroll
                        for (int c = 0; c < CPT / 2; ++c)
                            dv[u][c] = reinterpret_cast<const double2*>(d_t + (kb + U + u) * P)[c];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) acc[c] = __dadd_rn(acc[c], prod[u][c]);
            }
        } else {
            for (int kk = 0; kk < rows; ++kk) {
                const double a = a_t[kk * BR];
                const double2* d2 = reinterpret_cast<const double2*>(d_t + kk * P);
#pragma unroll
                for (int c = 0; c < CPT / 2; ++c) {
                    const double2 dv = d2[c];
                    acc[2 * c] = mac_exact(acc[2 * c], a, dv.x);
                    acc[2 * c + 1] = mac_exact(acc[2 * c + 1], a, dv.y);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) {
            s = 0;
            phase ^= 1u;
        }
    }

    const int il = i0 + r;
    if (il < n_loc && g < P / CPT) {
        const int row = row0 + il;
        const double bb = (b != nullptr) ? b[row] : 0.0;
        double v[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int col = g * CPT + c;
            v[c] = 0.0;
            if (col < p) v[c] = (b != nullptr) ? __dsub_rn(acc[c], bb) : acc[c];
        }
        const size_t o = static_cast<size_t>(row) * P + g * CPT;
        if (!PUSH) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) Y[o + c] = v[c];
        } else {
            for (int q = 0; q < peers.n; ++q)  // this rank's rows into every rank's copy
#pragma unroll
                for (int c = 0; c < CPT; ++c) peers.dst[q][o + c] = v[c];
        }
    }
    if (PUSH) __threadfence_system();
}

// Two rows per thread (RPT = 2, used at p >= 16): one 16-byte load of A
// serves both rows' chains.  Same arithmetic as ad_exact_kernel, kept as a
// separate kernel because the RPT = 1 case compiles ~5% slower inside this
// template (tools/probe/ad_cmp_probe.cu).
template <int P, int CPT, int BR, int T, int S, int RPT = 2, bool PUSH = false>
__global__ void __launch_bounds__(32 + 32 * ad_consumer_warps(BR / RPT, P / CPT))
    ad_exact_rpt_kernel(const double* __restrict__ Ap, int n, int n_loc, int row0,
                    const double* __restrict__ D, double* __restrict__ Y,
                    const double* __restrict__ b, int p, const int* __restrict__ stop, PeerRows peers,
                    int res_k) {
    pdl_wait();
    constexpr int RT = BR / RPT;  // row-threads per column group
    constexpr int kConsumerWarps = ad_consumer_warps(RT, P / CPT);
    static_assert(RPT == 1 || RPT == 2, "1 or 2 rows per thread");
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Ds = As + S * T * BR;
    uint64_t* full = reinterpret_cast<uint64_t*>(Ds + S * T * P);
    uint64_t* empty = full + S;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.x * BR;
    const int ntiles = (n + T - 1) / T;
    const double* panel = Ap + static_cast<size_t>(blockIdx.x) * n * BR;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // Producer: one lane streams the A panel tiles and the D tiles.
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy(), pol_res = l2_evict_last_policy();
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int k0 = t * T;
                const int rows = min(T, n - k0);
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows) * (BR * 8u + P * 8u));
                bulk_g2s_evict_first(As + s * T * BR, panel + static_cast<size_t>(k0) * BR,
                                     static_cast<uint32_t>(rows) * BR * 8u, &full[s], k0 < res_k ? pol_res : pol);
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
    const int r = tid % RT;   // this thread's rows: RPT * r .. RPT * r + RPT - 1
    const int g = tid / RT;  // == P / CPT for the surplus threads (no output)
    const int gl = min(g, P / CPT - 1);
    double acc[RPT][CPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[q][c] = 0.0;

    int s = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
        mbar_wait(&full[s], phase);
        const double* a_t = As + s * T * BR + RPT * r;
        const double* d_t = Ds + s * T * P + gl * CPT;
        const int rows = min(T, n - t * T);
        if (rows == T) {
            constexpr int U = (CPT * RPT >= 8) ? 2 : 4;
            static_assert(T % U == 0, "T must be a multiple of U");
            double av[U][RPT];
            double2 dv[U][CPT / 2];
            auto load = [&](int kk, int u) {
                if (RPT == 2) {
                    const double2 a2 = *reinterpret_cast<const double2*>(a_t + kk * BR);
                    av[u][0] = a2.x;
                    av[u][RPT - 1] = a2.y;
                } else {
                    av[u][0] = a_t[kk * BR];
                }
#pragma unroll
                for (int c = 0; c < CPT / 2; ++c) dv[u][c] = reinterpret_cast<const double2*>(d_t + kk * P)[c];
            };
#pragma unroll
            for (int u = 0; u < U; ++u) load(u, u);
#pragma unroll
            for (int kb = 0; kb < T; kb += U) {
                double prod[U][RPT][CPT];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < RPT; ++q)
#pragma unroll
                        for (int c = 0; c < CPT / 2; ++c) {
                            prod[u][q][2 * c] = __dmul_rn(av[u][q], dv[u][c].x);
                            prod[u][q][2 * c + 1] = __dmul_rn(av[u][q], dv[u][c].y);
                        }
                if (kb + U < T) {
#pragma unroll
                    for (int u = 0; u < U; ++u) load(kb + U + u, u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < RPT; ++q)
#pragma unroll
                        for (int c = 0; c < CPT; ++c) acc[q][c] = __dadd_rn(acc[q][c], prod[u][q][c]);
            }
        } else {
            for (int kk = 0; kk < rows; ++kk) {
                const double2* d2 = reinterpret_cast<const double2*>(d_t + kk * P);
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const double a = a_t[kk * BR + q];
#pragma unroll
                    for (int c = 0; c < CPT / 2; ++c) {
                        const double2 dv = d2[c];
                        acc[q][2 * c] = mac_exact(acc[q][2 * c], a, dv.x);
                        acc[q][2 * c + 1] = mac_exact(acc[q][2 * c + 1], a, dv.y);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) {
            s = 0;
            phase ^= 1u;
        }
    }

#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int il = i0 + RPT * r + q;
        if (il < n_loc && g < P / CPT) {
            const int row = row0 + il;
            const double bb = (b != nullptr) ? b[row] : 0.0;
            const size_t o = static_cast<size_t>(row) * P + g * CPT;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int col = g * CPT + c;
                double v = 0.0;
                if (col < p) v = (b != nullptr) ? __dsub_rn(acc[q][c], bb) : acc[q][c];
                if (!PUSH) {
                    Y[o + c] = v;
                } else {
                    for (int pr = 0; pr < peers.n; ++pr) peers.dst[pr][o + c] = v;
                }
            }
        }
    }
    if (PUSH) __threadfence_system();
}

// Pipelined variant (P = 8 / 16 at large n, P = 4 at small n): thread = RPT
// rows x CPT columns, operands software-pipelined two batches of U k-steps
// ahead in two register
// sets (the chain kernel's scheme below), one straight-line body per tile, a
// 3-stage ring (tile t+1 is waited for at the top of tile t).  Per warp and
// k-step: one LDS.128 of A (two rows) and two broadcast LDS.128 of D feed 16
// DMUL + 16 DADD, i.e. 8 shared-memory wavefronts per 256 MACs against 6 per
// 128 in ad_exact_kernel, whose doubly-loaded SMs are shared-memory bound
// (48 wavefronts vs 32 FP64-pipe cycles per k-step; profiles/).  One CTA of
// 4 consumer warps per SM (P = 8 with BR = 128, P = 16 with BR = 64): a CTA's
// warps map to SMSPs by warp index, so producer + 4 consumers keep one
// consumer warp per SMSP (two co-resident 2-warp CTAs would stack theirs on
// two SMSPs: 617 us in the probe).  tools/probe/ad_v3_probe.cu: n = 16384, P = 8:
// 349 us vs 422 us; n = 65536, P = 16: 10.0 ms vs 11.1 ms.  At P = 4 and
// n < 9472 (1 row x 2 columns, 32-row panels, 2 warps) a deeper ring keeps
// enough bytes in flight for the latency-bound small case: n = 4096 34 us vs
// 47 us.  Same arithmetic and order as ad_exact_kernel.
constexpr int kPipeU = 2;  // k-steps per batch (deeper batches measured no better)
__host__ __device__ constexpr size_t ad_pipe_smem(int P, int BR, int T, int S) {
    return static_cast<size_t>(S) * T * (BR + P) * sizeof(double) + 2 * S * sizeof(uint64_t);
}
template <int P, int CPT, int RPT, int BR, int T, int S, bool PUSH = false>
__global__ void __launch_bounds__(32 + 32 * ad_consumer_warps(BR / RPT, P / CPT))
    ad_exact_pipe_kernel(const double* __restrict__ Ap, int n, int n_loc, int row0,
                         const double* __restrict__ D, double* __restrict__ Y,
                         const double* __restrict__ b, int p, const int* __restrict__ stop, PeerRows peers,
                    int res_k) {
    pdl_wait();
    constexpr int U = kPipeU;
    static_assert(RPT == 1 || RPT == 2, "rows per thread");
    static_assert(CPT % 2 == 0, "columns per thread come in double2 pairs");
    constexpr int RG = BR / RPT;
    constexpr int NW = ad_consumer_warps(RG, P / CPT);
    constexpr int NBT = T / U;
    static_assert(T % (2 * U) == 0, "even number of batches per tile");
    static_assert((RG * (P / CPT)) % 32 == 0, "whole consumer warps");
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Ds = As + S * T * BR;
    uint64_t* full = reinterpret_cast<uint64_t*>(Ds + S * T * P);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (n + T - 1) / T;
    const double* panel = Ap + static_cast<size_t>(blockIdx.x) * n * BR;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy(), pol_res = l2_evict_last_policy();
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int k0 = t * T;
                const int rows = min(T, n - k0);
                mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(rows) * (BR * 8u + P * 8u));
                bulk_g2s_evict_first(As + s * T * BR, panel + static_cast<size_t>(k0) * BR,
                                     static_cast<uint32_t>(rows) * BR * 8u, &full[s], k0 < res_k ? pol_res : pol);
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
    const int rr = tid % RG, g = tid / RG;
    const int aoff = rr * RPT, doff = g * CPT;
    auto tile_wait = [&](int t) {
        if (t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    // batch j = k-steps j*U .. j*U+U-1: ring stage (j / NBT) % S.  Batches
    // past the last tile read stale ring data that is multiplied, never added.
    auto load = [&](int j, double (&a)[U][RPT], double (&d)[U][CPT]) {
        const int st = (j / NBT) % S, kk = (j % NBT) * U;
        const double* ab = As + st * T * BR + kk * BR + aoff;
        const double* db = Ds + st * T * P + kk * P + doff;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (RPT == 2) {
                const double2 av = *reinterpret_cast<const double2*>(ab + u * BR);
                a[u][0] = av.x;
                a[u][1] = av.y;
            } else {
                a[u][0] = ab[u * BR];
            }
#pragma unroll
            for (int c = 0; c < CPT / 2; ++c) {
                const double2 dv = reinterpret_cast<const double2*>(db + u * P)[c];
                d[u][2 * c] = dv.x;
                d[u][2 * c + 1] = dv.y;
            }
        }
    };
    double acc[RPT][CPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[r][c] = 0.0;
    double pr[U][RPT][CPT];
    double ae[U][RPT], ao[U][RPT], de[U][CPT], dq[U][CPT];
    // add batch b, form batch b+1 (read set), load batch b+2 (write set)
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
            // partial last tile: the batches that hold k-steps, the last masked
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
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int il = blockIdx.x * BR + aoff + r;
        if (il < n_loc) {
            const int row = row0 + il;
            const double bb = (b != nullptr) ? b[row] : 0.0;
            const size_t o = static_cast<size_t>(row) * P + doff;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                double v = 0.0;
                if (doff + c < p) v = (b != nullptr) ? __dsub_rn(acc[r][c], bb) : acc[r][c];
                if (!PUSH) {
                    Y[o + c] = v;
                } else {
                    for (int q = 0; q < peers.n; ++q) peers.dst[q][o + c] = v;
                }
            }
        }
    }
    if (PUSH) __threadfence_system();
}

// ---------------------------------------------------------------------------
// (2) Sequential dot-product chains: Gram rows, step right-hand sides and
// norms (block_cg.hpp:153-160, :214-216, :262-264, :275-276; kernels.hpp:20-26).
// Each chain is one thread walking k = 0..n-1 in order, acc = acc + x_k*y_k
// with both roundings kept: a dependent-DADD chain (8.5 cycles per DADD
// measured, tools/probe/clock_probe.cu).  Written naively, ptxas schedules
// DMUL(k) right before DADD(k) with the LDS of its operands just ahead, and
// each step pays the load, DMUL and DADD latencies (~16 cycles).  Here the
// chain is software-pipelined over batches of U rows: step b adds batch b's
// products (formed one step earlier), forms batch b+1's products and loads
// batch b+2's operands, alternating two operand register sets so that the
// loads never wait on the DMULs reading the other set.  One loop iteration
// covers a whole tile (straight-line steps, a single basic block for ptxas);
// tile t+1 is waited for at the top and tile t released at the bottom.
// Static issue cost ~10 cycles per step (tools/probe/chain_kernel_probe.cu).
//
// Tiles of T rows of up to three n x P row-major source blocks stream through
// an S-stage shared-memory ring: warp 0 is the producer (one lane issues the
// bulk copies, waiting on per-stage "empty" barriers); warps 1..2 run one
// chain per thread (64 chains per CTA) and release a stage with one
// (predicated) arrive per warp.
constexpr int kChainWarps = 2;
constexpr int kChainU = 16;  // rows per pipelined batch
constexpr int kChainThreads = 32 * (1 + kChainWarps);

__host__ __device__ constexpr size_t chain_smem_bytes(int P, int T, int S, int nsrc) {
    return static_cast<size_t>(S) * nsrc * T * P * sizeof(double) + 2 * S * sizeof(uint64_t);
}

template <int P, int T, int S>
__global__ void __launch_bounds__(kChainThreads)
    chain_kernel(const double* __restrict__ s0, const double* __restrict__ s1,
                 const double* __restrict__ s2, int nsrc, int n,
                 const ChainDesc* __restrict__ descs, int nchains, double* __restrict__ out,
                 const int* __restrict__ stop) {
    pdl_wait();
    constexpr int U = kChainU;
    static_assert(T % (2 * U) == 0, "tile rows must be an even number of batches");
    constexpr int NBT = T / U;  // batches per tile
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* buf = reinterpret_cast<double*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(buf + static_cast<size_t>(S) * nsrc * T * P);
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
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int t = 0; t < ntiles; ++t) {
                if (t >= S) mbar_wait(&empty[s], ph ^ 1u);
                const int rows = min(T, n - t * T);
                const uint32_t bytes = static_cast<uint32_t>(rows) * P * 8u;
                mbar_arrive_expect_tx(&full[s], bytes * nsrc);
                double* dst = buf + static_cast<size_t>(s) * nsrc * T * P;
                bulk_g2s(dst, s0 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 1) bulk_g2s(dst + T * P, s1 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (nsrc > 2) bulk_g2s(dst + 2 * T * P, s2 + static_cast<size_t>(t) * T * P, bytes, &full[s]);
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int c = blockIdx.x * (kChainWarps * 32) + (tid - 32);
    ChainDesc d{0, 0, 0, 0, 0, 0, 0};
    if (c < nchains) d = descs[c];
    const int xoff = d.sx * T * P + d.a;
    const int yoff = d.sy * T * P + d.b;
    const int nb = (n + U - 1) / U;  // batches; all full except possibly the last
    auto tile_wait = [&](int t) {
        if (t < ntiles) mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
    };
    // operands of batch j (may lie past the last tile: stale ring data that
    // is multiplied but never added)
    auto batch_base = [&](int j) -> const double* {
        return buf + static_cast<size_t>((j / NBT) % S) * nsrc * T * P + (j % NBT) * U * P;
    };
    double acc = 0.0;
    // pr: products of the batch being added; operands of batch j live in the
    // even (xe/ye) or odd (xo/yo) register set by the parity of j, so a step
    // reads one set and loads into the other (no WAR hazard to serialise the
    // loads behind the DMULs)
    double pr[U], xe[U], ye[U], xo[U], yo[U];
    // add batch b, form batch b+1 (from xr/yr), load batch b+2 (into xw/yw)
    auto step = [&](int b, const double (&xr)[U], const double (&yr)[U], double (&xw)[U], double (&yw)[U]) {
        const double* b2 = batch_base(b + 2);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc = __dadd_rn(acc, pr[u]);
            pr[u] = __dmul_rn(xr[u], yr[u]);
            xw[u] = b2[xoff + u * P];
            yw[u] = b2[yoff + u * P];
        }
    };
    tile_wait(0);
    {
        const double* b0 = batch_base(0);
        const double* b1 = batch_base(1);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pr[u] = __dmul_rn(b0[xoff + u * P], b0[yoff + u * P]);
            xo[u] = b1[xoff + u * P];
            yo[u] = b1[yoff + u * P];
        }
    }
    // One iteration per tile: tile t+1 is waited for first (the steps load up
    // to two batches ahead), the NBT steps run straight-line (one basic block
    // for ptxas to schedule), and tile t is released once its last batch has
    // been multiplied.
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
        tile_wait(t + 1);
        const int b0 = t * NBT;
        if ((t + 1) * T <= n) {
#pragma unroll
            for (int q = 0; q < NBT; q += 2) {
                step(b0 + q, xo, yo, xe, ye);
                step(b0 + q + 1, xe, ye, xo, yo);
            }
        } else {
            // partial last tile: the batches that hold rows, the last one masked
            for (int q = 0; q < NBT && b0 + q < nb; ++q) {
                const int b = b0 + q;
                if (b == nb - 1) {
                    const int rem = n - b * U;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < rem) acc = __dadd_rn(acc, pr[u]);
                } else if (q & 1) {
                    step(b, xe, ye, xo, yo);
                } else {
                    step(b, xo, yo, xe, ye);
                }
            }
        }
        __syncwarp();
        mbar_arrive_lane0(&empty[t % S], lane);
    }
    if (c < nchains) out[d.out] = d.neg ? -acc : acc;
}

// ---------------------------------------------------------------------------
// (3) Small p x p solves on one warp.
//
// lu_factor (kernels.hpp:61-95): partial pivoting, largest |.| with the
// lowest row index on ties; fails when the pivot is not above
// floor = max|M| * 1e-14 (block_cg.hpp:180-190).  Lane i owns row i during
// elimination; every element sees the reference's update sequence.
// lu_solve_vec (kernels.hpp:97-115): lane i solves agent i's row.
// Pivot search with the reference's sequential semantics
// (`if (cand > best)` scanning i = k+1.. from best = |a_kk|): the first index
// holding the maximum non-NaN value; a NaN at the diagonal always fails.
// Only lanes < P hold rows, so log2(P) xor-rounds reduce the maximum; the
// lowest lane holding it comes from a ballot (ties -> lowest index).
template <int P>
__device__ __forceinline__ int warp_pivot(double cand, int lane, int k, int p, bool* ok, double floor) {
    const bool elig = lane >= k && lane < p;
    const double v = (elig && !isnan(cand)) ? cand : -1.0;
    double vmax = v;
#pragma unroll
    for (int off = P / 2; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, vmax, off);
        vmax = (ov > vmax) ? ov : vmax;
    }
    vmax = __shfl_sync(0xffffffffu, vmax, 0);
    int idx = __ffs(__ballot_sync(0xffffffffu, elig && v == vmax)) - 1;
    const double diag = __shfl_sync(0xffffffffu, cand, k);
    const double best = isnan(diag) ? diag : vmax;
    if (isnan(diag)) idx = k;
    *ok = (best > floor);
    return idx;
}

// LU factorisation with lane i < p holding row i of M in registers (P is the
// compile-time bound, p <= P the active size).  Row exchanges and the pivot
// row broadcast are warp shuffles; each element sees the reference's update
// sequence a_ij = a_ij - mult * a_kj (kernels.hpp:61-95).  pv is the
// permutation entry of this lane's position.  Returns false on a pivot at or
// below the floor (uniform across the warp).
template <int P>
__device__ __forceinline__ bool lu_factor_regs(double (&m)[P], int& pv, int lane, int p, double floor) {
    pv = lane;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (k >= p) break;
        const double cand = (lane < p) ? fabs(m[k]) : 0.0;
        bool ok;
        const int piv = warp_pivot<P>(cand, lane, k, p, &ok, floor);
        if (!ok) return false;
        if (piv != k) {
            const int src = (lane == k) ? piv : ((lane == piv) ? k : lane);
#pragma unroll
            for (int j = 0; j < P; ++j) m[j] = __shfl_sync(0xffffffffu, m[j], src);
            pv = __shfl_sync(0xffffffffu, pv, src);
        }
        double rk[P];
#pragma unroll
        for (int j = 0; j < P; ++j) rk[j] = __shfl_sync(0xffffffffu, m[j], k);
        if (lane > k && lane < p) {
            const double mult = __ddiv_rn(m[k], rk[k]);
            m[k] = mult;
#pragma unroll
            for (int j = 0; j < P; ++j)
                if (j > k && j < p) m[j] = msub_exact(m[j], mult, rk[j]);
        }
    }
    return true;
}

// lu_solve_vec (kernels.hpp:97-115) for one right-hand side: forward
// y_i = rhs[perm_i] - sum_{j<i} L_ij y_j, backward
// x_i = (y_i - sum_{j>i} U_ij x_j) / U_ii, j ascending in both.
template <int P>
__device__ __forceinline__ void lu_solve_regs(const double (*lu)[P + 1], const int* perm, int p, const double* rhs,
                                              double (&x)[P]) {
    double y[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        y[i] = 0.0;
        x[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        if (i < p) {
            double acc = rhs[perm[i]];
#pragma unroll
            for (int j = 0; j < i; ++j) acc = msub_exact(acc, lu[i][j], y[j]);
            y[i] = acc;
        }
    }
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
        if (i < p) {
            double acc = y[i];
#pragma unroll
            for (int j = i + 1; j < P; ++j)
                if (j < p) acc = msub_exact(acc, lu[i][j], x[j]);
            x[i] = __ddiv_rn(acc, lu[i][i]);
        }
    }
}

// The two solves run inside the elementwise kernels that consume their
// coefficients: warp 0 of every CTA recomputes the (tiny, deterministic) p x p
// solve into shared memory while the other warps stage the CTA's first tile of
// operands, so a solve costs its latency once, not a launch plus a ramp.  All
// CTAs read the same inputs and run the same operation sequence, so they reach
// the same coefficients and the same stop decision; CTA 0 ("leader") alone
// writes the control block, the trace and the small-buffer copies.

// stage_gram_finalize + stage_alpha (block_cg.hpp:165-218) on one warp.
// alpha (row i = agent i) goes to coef[i * (P + 1) + j].  Returns false when
// the iteration stops (stop already set, SPD violation, rank collapse).
template <int P>
__device__ bool alpha_solve_warp(double* __restrict__ small, Ctl* ctl, double* coef, bool leader) {
    __shared__ double lu[P][P + 1];
    __shared__ double rh[P][P + 1];
    __shared__ int perm[P];
    const int lane = threadIdx.x;
    const SmallLayout L{P};
    const double* raw = small + L.raw();
    // Every input is requested up front (L2-coherent loads; griddepcontrol.wait
    // made the producers' writes visible), before the control fields resolve.
    const int stop = __ldcg(&ctl->stop);
    const int p = __ldcg(&ctl->p);
    double rr[P], rc[P], nsq = 0.0;
    if (lane < P) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            rr[j] = __ldcg(raw + lane * P + j);
            rc[j] = __ldcg(raw + j * P + lane);
            rh[lane][j] = __ldcg(small + L.rhs_a() + lane * P + j);
        }
        nsq = __ldcg(small + L.nsq_d() + lane);
    }
    if (stop) return false;
    // M(i,j) = (raw(i,j) + raw(j,i)) / 2.0 (x * 0.5 is the same rounding)
    double m[P];
    double maxabs = 0.0, diag = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) m[j] = 0.0;
    if (lane < p) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            if (j < p) {
                m[j] = __dmul_rn(__dadd_rn(rr[j], rc[j]), 0.5);
                const double a = fabs(m[j]);
                maxabs = (maxabs < a) ? a : maxabs;
                if (j == lane) diag = m[j];
            }
        }
    } else {
        nsq = 0.0;
    }
    // std::max over all entries ignores NaN in this formulation; order-free.
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, maxabs, off);
        maxabs = (maxabs < o) ? o : maxabs;
    }
    const double floor = __dmul_rn(maxabs, 1e-14);
    // SPD guard (block_cg.hpp:196-202): nonpositive d_i^T A d_i with d_i != 0.
    const bool bad = (lane < p) && !(diag > 0.0) && (nsq > 0.0);
    if (__any_sync(0xffffffffu, bad)) {
        if (leader && lane == 0) {
            ctl->err = 2;  // COOPCG_E_SPD_VIOLATION
            ctl->err_iter = ctl->k;
            ctl->stop = 1;
        }
        return false;
    }
    int pv;
    if (!lu_factor_regs<P>(m, pv, lane, p, floor)) {
        if (leader && lane == 0) {
            // RankCollapse (solvers.hpp:117-123); steepest descent reports a
            // vanished gradient energy with r = 0 as Converged (solvers.hpp:588-594)
            ctl->status = (ctl->algo == 2) ? 0 : 1;
            if (ctl->algo == 2) ctl->converged_agent = 0;
            ctl->stop = 1;
        }
        return false;
    }
    if (lane < P) {
#pragma unroll
        for (int j = 0; j < P; ++j) lu[lane][j] = m[j];
        perm[lane] = pv;
    }
    __syncwarp();
    if (lane < p) {
        double x[P];
        lu_solve_regs<P>(lu, perm, p, rh[lane], x);
#pragma unroll
        for (int j = 0; j < P; ++j) coef[lane * (P + 1) + j] = x[j];
        if (leader) {
#pragma unroll
            for (int j = 0; j < P; ++j) small[L.alpha() + lane * P + j] = (j < p) ? x[j] : 0.0;
            // keep the factorisation for the beta solve (same M, same pivots)
#pragma unroll
            for (int j = 0; j < P; ++j) ctl->lu[lane * P + j] = m[j];
            ctl->perm[lane] = pv;
        }
    }
    return true;
}

// stage_beta (block_cg.hpp:248-266) + the norms of stage_direction_and_norms
// (:275-276) + the record / convergence part of end_of_iteration
// (solvers.hpp:125-154) on one warp.  beta goes to coef; returns false when
// the iteration stops (stop already set, or an agent converged).
template <int P>
__device__ bool beta_solve_warp(double* __restrict__ small, Ctl* ctl, double* coef, bool leader,
                                double* __restrict__ tr_norms, double* __restrict__ tr_minres,
                                unsigned long long* __restrict__ tr_wall, int capacity) {
    __shared__ double lu[P][P + 1];
    __shared__ double rh[P][P + 1];
    __shared__ int perm[P];
    __shared__ double norms[P];
    const int lane = threadIdx.x;
    const SmallLayout L{P};
    const int stop = __ldcg(&ctl->stop);
    const int p = __ldcg(&ctl->p);
    const int algo = __ldcg(&ctl->algo);
    const double tol = __ldcg(&ctl->tol);
    double nsq = 0.0;
    if (lane < P) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            lu[lane][j] = __ldcg(&ctl->lu[lane * P + j]);
            rh[lane][j] = __ldcg(small + L.rhs_b() + lane * P + j);
        }
        perm[lane] = __ldcg(&ctl->perm[lane]);
        nsq = __ldcg(small + L.nsq_r() + lane);
    }
    if (stop) return false;
    __syncwarp();
    if (lane < p) {
        double x[P];
        if (algo == 2) {  // steepest descent: D' = R (no conjugation)
#pragma unroll
            for (int j = 0; j < P; ++j) x[j] = 0.0;
        } else {
            lu_solve_regs<P>(lu, perm, p, rh[lane], x);
        }
#pragma unroll
        for (int j = 0; j < P; ++j) coef[lane * (P + 1) + j] = x[j];
        norms[lane] = __dsqrt_rn(nsq);
        if (leader) {
#pragma unroll
            for (int j = 0; j < P; ++j) small[L.beta() + lane * P + j] = (j < p) ? x[j] : 0.0;
            small[L.norm() + lane] = norms[lane];
        }
    }
    __syncwarp();
    // first agent at or below the tolerance (block_cg.hpp:297-303); every CTA
    // computes it from the same norms
    int slot = -1;
    for (int j = 0; j < p; ++j)
        if (slot < 0 && norms[j] <= tol) slot = j;
    if (leader) {
        const int k = ctl->k;
        const int p0 = ctl->p0;
        if (k < capacity) {
            // per-original-id record; ids that left the block (mccg) stay NaN
            for (int j = lane; j < p0; j += 32)
                tr_norms[static_cast<size_t>(k) * p0 + j] = __longlong_as_double(0x7ff8000000000000ll);
            __syncwarp();
            if (lane < p) tr_norms[static_cast<size_t>(k) * p0 + ctl->ids[lane]] = norms[lane];
        }
        if (lane == 0) {
            const unsigned long long now = globaltimer_ns();
            double mn = norms[0];
            for (int j = 0; j < p; ++j) mn = (norms[j] < mn) ? norms[j] : mn;  // std::min
            if (k < capacity) {
                tr_minres[k] = mn;
                tr_wall[k] = now - ctl->t_last;
            }
            ctl->t_last = now;
            ctl->iterations = k + 1;
            if (slot >= 0) {
                ctl->status = 0;  // Converged
                ctl->converged_agent = ctl->ids[slot];
                ctl->stop = 1;
            }
        }
    }
    return slot < 0;
}

// ---------------------------------------------------------------------------
// (4) Elementwise block updates (kernels.hpp:36-49 combine_columns:
// dest = base + sum_j coeff[j] * B(:, j), j ascending).  One thread per
// (row, agent) element; a CTA step covers kUpdTiles tiles of 256 elements
// (256 / P rows each) whose operands are staged in shared memory (coalesced:
// thread t loads element t of each tile), so each thread keeps kUpdTiles
// loads per operand in flight even when the solve's registers allow only one
// CTA per SM.
//
// alpha_update_kernel (alpha solve + block_cg.hpp:218-244):
//   mode 0: R_i += sum_j alpha_ij Q_j ; X_i += sum_j alpha_ij D_j (recurrence)
//   mode 1: X_i += sum_j alpha_ij D_j only (recompute iterations: R is then
//           recomputed as A X - b by ad_exact_kernel; block_cg.hpp:222-244)
constexpr int kUpdTiles = 4;
template <int P>
__global__ void __launch_bounds__(256)
    alpha_update_kernel(double* __restrict__ R, double* __restrict__ X, const double* __restrict__ Q,
                        const double* __restrict__ D, double* __restrict__ small, int n, int p, int mode, Ctl* ctl) {
    pdl_wait();
    constexpr int U = kUpdTiles;
    __shared__ double coef[P * (P + 1)];
    __shared__ double tq[U * 256], td[U * 256];
    __shared__ int go;
    const int tid = threadIdx.x;
    const int i = tid % P;
    const int nel = n * P;
    const int nblk = (nel + U * 256 - 1) / (U * 256);
    double r[U], x[U];
    auto stage = [&](int blk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = (blk * U + u) * 256 + tid;
            if (e < nel) {
                if (mode == 0) {
                    tq[u * 256 + tid] = Q[e];
                    r[u] = R[e];
                }
                td[u * 256 + tid] = D[e];
                x[u] = X[e];
            }
        }
    };
    int blk = blockIdx.x;
    if (blk < nblk) stage(blk);
    if (tid < 32) {
        const bool ok = alpha_solve_warp<P>(small, ctl, coef, blockIdx.x == 0);
        if (tid == 0) go = ok;
    }
    __syncthreads();
    if (!go) return;
    const double* a = coef + i * (P + 1);
    const int rl = tid - i;  // first element of this thread's row in a tile
    while (blk < nblk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = (blk * U + u) * 256 + tid;
            if (e < nel && i < p) {
                if (mode == 0) {
                    double acc = r[u];
                    for (int j = 0; j < p; ++j) acc = mac_exact(acc, a[j], tq[u * 256 + rl + j]);
                    R[e] = acc;
                }
                double acc = x[u];
                for (int j = 0; j < p; ++j) acc = mac_exact(acc, a[j], td[u * 256 + rl + j]);
                X[e] = acc;
            }
        }
        blk += gridDim.x;
        if (blk >= nblk) break;
        __syncthreads();
        stage(blk);
        __syncthreads();
    }
}

// Pairs (i <= j < p) of the Gram Dn^T Dn handled by thread tid (up to 3).
__device__ __forceinline__ void gram_pairs(int tid, int p, int (&pi)[3], int (&pj)[3]) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        int t = tid + q * 256;
        pi[q] = -1;
        pj[q] = -1;
        if (t < p * (p + 1) / 2) {
            int i = 0;
            while (t >= p - i) {
                t -= p - i;
                ++i;
            }
            pi[q] = i;
            pj[q] = i + t;
        }
    }
}

// Accumulate `rows` staged rows (tile[], row-major, stride P) into the pair
// partials: fast (reordered, FMA) sums, used only by the rank certificate.
template <int P>
__device__ __forceinline__ void gram_tile(const double* tile, int rows, const int (&pi)[3], const int (&pj)[3],
                                          double (&part)[3]) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        if (pi[q] >= 0) {
            double s = part[q];
            for (int rr = 0; rr < rows; ++rr) s = fma(tile[rr * P + pi[q]], tile[rr * P + pj[q]], s);
            part[q] = s;
        }
    }
}

// beta solve + record, then Dn = R + D beta^T (block_cg.hpp:270-273; D' = R
// for steepest descent, sd_copy) plus per-CTA partial Grams of Dn for the
// rank certificate (rank_end_kernel sums gridDim.x partials).  Same staging
// as alpha_update_kernel.
template <int P>
__global__ void __launch_bounds__(256)
    beta_direction_kernel(const double* __restrict__ R, const double* __restrict__ D, double* __restrict__ Dn,
                          double* __restrict__ small, int n, int p, double* __restrict__ partials, Ctl* ctl,
                          double* __restrict__ tr_norms, double* __restrict__ tr_minres,
                          unsigned long long* __restrict__ tr_wall, int capacity, int sd_copy) {
    pdl_wait();
    constexpr int U = kUpdTiles;
    __shared__ double coef[P * (P + 1)];
    __shared__ double td[U * 256], tile[U * 256];
    __shared__ int go;
    const int tid = threadIdx.x;
    const int i = tid % P;
    const int nel = n * P;
    const int nblk = (nel + U * 256 - 1) / (U * 256);
    double r[U];
    auto stage = [&](int blk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = (blk * U + u) * 256 + tid;
            if (e < nel) {
                r[u] = R[e];
                td[u * 256 + tid] = D[e];
            }
        }
    };
    int blk = blockIdx.x;
    if (blk < nblk) stage(blk);
    if (tid < 32) {
        const bool ok = beta_solve_warp<P>(small, ctl, coef, blockIdx.x == 0, tr_norms, tr_minres, tr_wall, capacity);
        if (tid == 0) go = ok;
    }
    int pi[3], pj[3];
    double part[3] = {0.0, 0.0, 0.0};
    gram_pairs(tid, p, pi, pj);
    __syncthreads();
    if (!go) return;
    const double* a = coef + i * (P + 1);
    const int rl = tid - i;
    while (blk < nblk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = (blk * U + u) * 256 + tid;
            double v = 0.0;
            if (e < nel) {
                if (i < p) {
                    double acc = r[u];
                    if (!sd_copy)
                        for (int j = 0; j < p; ++j) acc = mac_exact(acc, a[j], td[u * 256 + rl + j]);
                    v = acc;
                }
                Dn[e] = v;
            }
            tile[u * 256 + tid] = v;
        }
        __syncthreads();
        gram_tile<P>(tile, U * (256 / P), pi, pj, part);
        blk += gridDim.x;
        if (blk < nblk) stage(blk);
        __syncthreads();
    }
    const int npairs = p * (p + 1) / 2;
#pragma unroll
    for (int q = 0; q < 3; ++q)
        if (pi[q] >= 0) partials[static_cast<size_t>(blockIdx.x) * npairs + tid + q * 256] = part[q];
}

// Partial Grams of an existing direction block (setup: D0 = R0; the
// kernel-level rank entry point).  Same tiling and sums as above.
template <int P>
__global__ void __launch_bounds__(256)
    gram_partials_kernel(const double* __restrict__ D, int n, int p, double* __restrict__ partials,
                         const int* __restrict__ stop) {
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    __shared__ double tile[256];
    const int tid = threadIdx.x;
    const int i = tid % P;
    constexpr int kRows = 256 / P;
    const int ntiles = (n + kRows - 1) / kRows;
    int pi[3], pj[3];
    double part[3] = {0.0, 0.0, 0.0};
    gram_pairs(tid, p, pi, pj);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int row = t * kRows + tid / P;
        tile[tid] = (row < n && i < p) ? D[static_cast<size_t>(row) * P + i] : 0.0;
        __syncthreads();
        gram_tile<P>(tile, kRows, pi, pj, part);
        __syncthreads();
    }
    const int npairs = p * (p + 1) / 2;
#pragma unroll
    for (int q = 0; q < 3; ++q)
        if (pi[q] >= 0) partials[static_cast<size_t>(blockIdx.x) * npairs + tid + q * 256] = part[q];
}

// ---------------------------------------------------------------------------
// (5) Rank check of the direction block (solvers.hpp:156-162 calls
// numerical_rank(Dnext, rank_rel_tol), dense_ops.hpp:104-157) and the rest of
// end_of_iteration.  A certificate first: from G = Dn^T Dn (fast partials),
// normalise to unit diagonal, Cholesky, and bound lambda_min(G^) >=
// 1/||L^-1||_F^2.  Every pivot of column-pivoted MGS is >= sigma_min(Dn)^2 >=
// lambda_min(G^) * min_j G_jj while the first pivot is max_j G_jj, so if
// lambda_lower * min/max clears the rank tolerance by a wide margin MGS
// reports full rank.  Otherwise the exact MGS restatement runs (same op order
// as the reference) and its rank is used.  One CTA of 1024 threads.
struct RankScratch {
    double g[kMaxP][kMaxP + 1];
    double l[kMaxP][kMaxP + 1];
    double wi[kMaxP][kMaxP + 1];
    double vals[kMaxP];
    double coefs[kMaxP];
    int used[kMaxP];
    int ok;
    int best;
    double best_sq;
    int rank;
    int brk;
};

template <int T>
__device__ void cta_exact_chains(const double* __restrict__ V, int n, int P, int nact, const int* xcol,
                                 const int* ycol, double* outv, double* buf, uint64_t* bar, int& phase_ctr) {
    // Chains: thread c < nact computes sum_k V[k][xcol[c]] * V[k][ycol[c]].
    const int tid = threadIdx.x;
    const int ntiles = (n + T - 1) / T;
    double acc = 0.0;
    const int xc = (tid < nact) ? xcol[tid] : 0;
    const int yc = (tid < nact) ? ycol[tid] : 0;
    auto issue = [&](int t) {
        if (tid == 0) {
            const int rows = min(T, n - t * T);
            const uint32_t bytes = static_cast<uint32_t>(rows) * P * 8u;
            const int slot = (phase_ctr + t) & 1;
            mbar_arrive_expect_tx(&bar[slot], bytes);
            bulk_g2s(buf + slot * T * P, V + static_cast<size_t>(t) * T * P, bytes, &bar[slot]);
        }
    };
    issue(0);
    for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) issue(t + 1);
        const int use = phase_ctr + t;
        mbar_wait(&bar[use & 1], static_cast<uint32_t>(use >> 1) & 1u);
        if (tid < nact) {
            const double* tl = buf + (use & 1) * T * P;
            const int rows = min(T, n - t * T);
            for (int kk = 0; kk < rows; ++kk) acc = mac_exact(acc, tl[kk * P + xc], tl[kk * P + yc]);
        }
        __syncthreads();
    }
    phase_ctr += ntiles;
    if (tid < nact) outv[tid] = acc;
    __syncthreads();
}

constexpr int kRankTile = 64;

// mode 0: end of iteration k; mode 1: setup (rank of D0, then max_iters==0);
// mode 2: rank only (kernel-level entry point).
__global__ void __launch_bounds__(1024)
    rank_end_kernel(const double* __restrict__ partials, int nparts, const double* __restrict__ Dn,
                    double* __restrict__ V, int n, Ctl* ctl, int mode, double* __restrict__ small_out) {
    pdl_wait();
    if (*reinterpret_cast<volatile int*>(&ctl->stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int p = ctl->p, P = ctl->P;
    double* buf = reinterpret_cast<double*>(smem_raw);  // 2 * kRankTile * P
    uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 2 * kRankTile * P);
    __shared__ RankScratch rs;
    __shared__ int xcol[kMaxP], ycol[kMaxP];
    const int tid = threadIdx.x;
    const int npairs = p * (p + 1) / 2;
    // 1. fixed-order reduction of the partial Grams (pairs i <= j).
    {
        __shared__ double red[1024], pv[kMaxP * (kMaxP + 1) / 2];
        cta_reduce_fixed(partials, nparts, npairs, 0, 1, npairs, pv, red);
        for (int qq = tid; qq < npairs; qq += blockDim.x) {
            int t = qq, i = 0;
            while (t >= p - i) {
                t -= p - i;
                ++i;
            }
            rs.g[i][i + t] = pv[qq];
            rs.g[i + t][i] = pv[qq];
        }
        __syncthreads();
    }
    // The next iteration's |D_i|^2 (fast mode's SPD-guard input; the exact
    // path recomputes it with an exact chain).
    if (small_out != nullptr && tid < p) small_out[SmallLayout{P}.nsq_d() + tid] = rs.g[tid][tid];
    // 2. certificate on warp 0
    if (tid < 32) {
        const int lane = tid;
        double dmin = 0, dmax = 0;
        bool good = true;
        for (int j = 0; j < p; ++j) {
            const double dj = rs.g[j][j];
            if (!(dj > 0.0) || !isfinite(dj)) good = false;
            if (j == 0 || dj < dmin) dmin = dj;
            if (j == 0 || dj > dmax) dmax = dj;
        }
        if (good) {
            // sqrt(g_ii) * sqrt(g_jj): the product g_ii * g_jj underflows in the
            // post-convergence tail (entries ~1e-80, Gram ~1e-160).
            if (lane < p)
                for (int j = 0; j < p; ++j)
                    rs.l[lane][j] = rs.g[lane][j] / (sqrt(rs.g[lane][lane]) * sqrt(rs.g[j][j]));
            __syncwarp();
            // Cholesky, lane owns row
            for (int k = 0; k < p && good; ++k) {
                if (lane == k) {
                    double s = rs.l[k][k];
                    for (int m = 0; m < k; ++m) s -= rs.l[k][m] * rs.l[k][m];
                    rs.vals[k] = (s > 0.0 && isfinite(s)) ? sqrt(s) : -1.0;
                    rs.l[k][k] = rs.vals[k];
                }
                __syncwarp();
                if (!(rs.vals[k] > 0.0)) good = false;
                if (good && lane > k && lane < p) {
                    double s = rs.l[lane][k];
                    for (int m = 0; m < k; ++m) s -= rs.l[lane][m] * rs.l[k][m];
                    rs.l[lane][k] = s / rs.l[k][k];
                }
                __syncwarp();
            }
            double fro = 0.0;
            if (good && lane < p) {
                // column `lane` of L^-1
                const int j = lane;
                for (int i = 0; i < p; ++i) rs.wi[i][j] = 0.0;
                rs.wi[j][j] = 1.0 / rs.l[j][j];
                fro = rs.wi[j][j] * rs.wi[j][j];
                for (int i = j + 1; i < p; ++i) {
                    double s = 0.0;
                    for (int m = j; m < i; ++m) s += rs.l[i][m] * rs.wi[m][j];
                    rs.wi[i][j] = -s / rs.l[i][i];
                    fro += rs.wi[i][j] * rs.wi[i][j];
                }
            }
            for (int off = 16; off > 0; off >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, off);
            if (good) {
                const double lam_lower = 1.0 / fro;
                const double tol = ctl->rank_rel_tol;
                // Every MGS pivot^2 >= lambda_min(G^) * min_j G_jj and the first
                // pivot^2 = max_j G_jj; MGS accepts while pivot^2 > tol^2 * first.
                // Demand lambda_lower(G^) > 1e-6 (well above the ~n*eps error of
                // the reordered Gram) and a 1e4 margin over tol^2.
                good = isfinite(lam_lower) && lam_lower > 1e-6 &&
                       lam_lower * (dmin / dmax) > tol * tol * 1e4 && dmin > 1e-280;
            }
        }
        if (lane == 0) rs.ok = good ? 1 : 0;
    }
    __syncthreads();
    int rank = p;
    if (!rs.ok || ctl->force_exact) {
        // 3. exact column-pivoted MGS (dense_ops.hpp:104-157) on a working copy.
        if (tid == 0) {
            ctl->exact_rank_checks += 1;
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            fence_mbar_init();
        }
        const size_t total = static_cast<size_t>(n) * P;
        for (size_t e = tid; e < total; e += blockDim.x) V[e] = Dn[e];
        if (tid < kMaxP) rs.used[tid] = 0;
        if (tid == 0) rs.rank = 0;
        __threadfence_block();
        __syncthreads();
        int phase_ctr = 0;
        double max_pivot_sq = 0.0;
        const double tol = ctl->rank_rel_tol;
        const double tol_sq = __dmul_rn(tol, tol);
        for (int step = 0; step < p; ++step) {
            // squared norms of unused columns
            if (tid == 0) {
                int a = 0;
                for (int j = 0; j < p; ++j)
                    if (!rs.used[j]) {
                        xcol[a] = j;
                        ycol[a] = j;
                        ++a;
                    }
                rs.best = a;  // temporarily: number of active chains
            }
            __syncthreads();
            const int nact = rs.best;
            __syncthreads();
            // make V writes visible to the async (bulk copy) proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncthreads();
            cta_exact_chains<kRankTile>(V, n, P, nact, xcol, ycol, rs.vals, buf, bar, phase_ctr);
            if (tid == 0) {
                int best = -1;
                double best_sq = 0.0;
                for (int a = 0; a < nact; ++a) {
                    const double nsq = rs.vals[a];
                    if (best < 0 || nsq > best_sq) {
                        best = xcol[a];
                        best_sq = nsq;
                    }
                }
                if (step == 0) max_pivot_sq = best_sq;
                rs.brk = !(best_sq > __dmul_rn(tol_sq, max_pivot_sq));
                if (!rs.brk) {
                    rs.used[best] = 1;
                    ctl->rank_cols[rs.rank] = best;
                    rs.rank += 1;
                }
                rs.best = best;
                rs.best_sq = best_sq;
            }
            __syncthreads();
            if (rs.brk) break;
            // projections: coef_j = dot(q, c_j) / qsq for unused j
            const int qb = rs.best;
            const double qsq = rs.best_sq;
            if (tid == 0) {
                int a = 0;
                for (int j = 0; j < p; ++j)
                    if (!rs.used[j]) {
                        xcol[a] = qb;
                        ycol[a] = j;
                        ++a;
                    }
                rs.brk = a;
            }
            __syncthreads();
            const int nproj = rs.brk;
            __syncthreads();
            if (nproj == 0) break;
            cta_exact_chains<kRankTile>(V, n, P, nproj, xcol, ycol, rs.vals, buf, bar, phase_ctr);
            if (tid < nproj) rs.coefs[tid] = __ddiv_rn(rs.vals[tid], qsq);
            __syncthreads();
            // c[i] -= coef * q[i]
            for (size_t e = tid; e < static_cast<size_t>(n) * nproj; e += blockDim.x) {
                const int a = static_cast<int>(e % nproj);
                const size_t row = e / nproj;
                const int j = ycol[a];
                V[row * P + j] = msub_exact(V[row * P + j], rs.coefs[a], V[row * P + qb]);
            }
            __threadfence_block();
            __syncthreads();
            if (tid == 0) rs.brk = 0;
            __syncthreads();
        }
        rank = rs.rank;
    }
    if (tid == 0) {
        ctl->rank_result = rank;
        if (mode == 0) {
            if (rank < p && ctl->algo == 2) {
                // steepest descent has no rank check: r = 0 ends with Converged
                // at the next gradient-energy test (solvers.hpp:588-594)
                ctl->status = 0;
                ctl->converged_agent = 0;
                ctl->stop = 1;
            } else if (rank < p && ctl->algo == 1) {
                // mccg (solvers.hpp:162-175): pause; the host selects the
                // surviving columns from numerical_rank(R), compacts and resumes.
                ctl->restrict_pending = 1;
                ctl->stop = 1;
            } else if (rank < p) {
                ctl->status = 1;  // RankCollapse (solvers.hpp:157-161)
                ctl->stop = 1;
            } else if (ctl->k + 1 >= ctl->max_iters) {
                ctl->status = 2;  // MaxIterations (solvers.hpp:177-181)
                ctl->stop = 1;
            } else {
                ctl->k += 1;
            }
        } else if (mode == 1) {
            if (ctl->algo == 1) {
                // mccg: the host applies setup_coordinator's restriction and
                // tolerance logic (solvers.hpp:63-98) after reading rank/columns.
                ctl->restrict_pending = 1;
            } else if (rank < p && ctl->algo == 2) {
                ctl->status = 0;  // steepest descent: zero gradient -> Converged (solvers.hpp:588-594)
                ctl->converged_agent = 0;
                ctl->stop = 1;
            } else if (rank < p) {
                ctl->status = 1;  // setup_coordinator, solvers.hpp:83-85
                ctl->stop = 1;
            } else if (ctl->max_iters == 0) {
                ctl->status = 2;  // solvers.hpp:95-98
                ctl->stop = 1;
            }
            ctl->t_last = globaltimer_ns();
        }
    }
}

// Setup coordinator part 1 (solvers.hpp:55-82): initial norms, minres and
// the tolerance check.  One warp.
__global__ void setup_norms_kernel(double* __restrict__ small, Ctl* ctl, double* __restrict__ init_norms) {
    const int lane = threadIdx.x;
    const int p = ctl->p;
    const SmallLayout L{ctl->P};
    if (lane < p) {
        const double v = __dsqrt_rn(small[L.nsq_r() + lane]);
        small[L.norm() + lane] = v;
        init_norms[lane] = v;
    }
    __syncwarp();
    if (lane == 0) {
        const double* nv = small + L.norm();
        double m = nv[0];
        int slot = -1;
        for (int j = 0; j < p; ++j) {
            m = (nv[j] < m) ? nv[j] : m;
            if (slot < 0 && nv[j] <= ctl->tol) slot = j;
        }
        init_norms[p] = m;
        if (slot >= 0 && ctl->algo == 0) {
            ctl->status = 0;
            ctl->converged_agent = slot;
            ctl->stop = 1;
        }
        ctl->t_last = globaltimer_ns();
    }
}

// mccg column compaction (BlockCgWorkspace::restrict_to, block_cg.hpp:84-96):
// new[:, c] = old[:, keep[c]] for c < pk, zero beyond.  One thread per row.
struct KeepList {
    int keep[kMaxP];
};
__global__ void compact_columns_kernel(double* __restrict__ blk, int n, int P, KeepList kl, int pk) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    double v[kMaxP];
    double* r = blk + static_cast<size_t>(row) * P;
    for (int c = 0; c < pk; ++c) v[c] = r[kl.keep[c]];
    for (int c = 0; c < P; ++c) r[c] = (c < pk) ? v[c] : 0.0;
}

// finalize_trace (solvers.hpp:188-210): final_residual_norms = ||A x_j - b||.
__global__ void final_norms_kernel(const double* __restrict__ small, const Ctl* ctl, double* __restrict__ out) {
    const int lane = threadIdx.x;
    const int p = ctl->p;
    const SmallLayout L{ctl->P};
    if (lane < p) out[lane] = __dsqrt_rn(small[L.nsq_f() + lane]);
    __syncwarp();
    if (lane == 0) {
        double m = out[0];
        for (int j = 1; j < p; ++j) m = (out[j] < m) ? out[j] : m;  // std::min_element
        out[p] = m;
    }
}

// ---------------------------------------------------------------------------
// Layout helpers.
// host DenseBlock (n x p column-major) <-> device row-major n x P, zero padded.
__global__ void colmajor_to_rowmajor_kernel(const double* __restrict__ src, double* __restrict__ dst, int n,
                                            int p, int P) {
    const size_t total = static_cast<size_t>(n) * P;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(e % P);
        const size_t k = e / P;
        dst[e] = (j < p) ? src[static_cast<size_t>(j) * n + k] : 0.0;
    }
}
__global__ void rowmajor_to_colmajor_kernel(const double* __restrict__ src, double* __restrict__ dst, int n,
                                            int p, int P) {
    const size_t total = static_cast<size_t>(n) * p;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t k = e % n;
        const int j = static_cast<int>(e / n);
        dst[e] = src[k * P + j];
    }
}
// rows [c0, c0+rows) of a row-major n-wide matrix (staging) -> panels.
__global__ void transpose_rows_kernel(const double* __restrict__ stage, int rows, int n, double* __restrict__ Ap,
                                      ALay L, int c0) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32;  // k
    const int by = blockIdx.y * 32;  // local row
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int i = by + yy, k = bx + threadIdx.x;
        tile[yy][threadIdx.x] = (i < rows && k < n) ? stage[static_cast<size_t>(i) * n + k] : 0.0;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int k = bx + yy, i = by + threadIdx.x;
        if (k < n && i < rows) Ap[a_idx(L, n, k, c0 + i)] = tile[threadIdx.x][yy];
    }
}
__global__ void untranspose_rows_kernel(const double* __restrict__ Ap, ALay L, int c0, int rows, int n,
                                        double* __restrict__ stage) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32;  // k
    const int by = blockIdx.y * 32;  // local row
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int k = bx + yy, i = by + threadIdx.x;
        tile[yy][threadIdx.x] = (k < n && i < rows) ? Ap[a_idx(L, n, k, c0 + i)] : 0.0;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int i = by + yy, k = bx + threadIdx.x;
        if (i < rows && k < n) stage[static_cast<size_t>(i) * n + k] = tile[threadIdx.x][yy];
    }
}

} // namespace coopcg_gpu
