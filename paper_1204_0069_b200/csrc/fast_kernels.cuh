// fast_kernels.cuh -- roofline ("fast") arithmetic mode of the cCG iteration.
//
// Same iteration as the reference (coopcg/block_cg.hpp:132-277) but with the
// floating-point work reordered for the hardware: FP64 tensor-core MMAs
// (mma.sync m8n8k4 .f64, SASS DMMA) for Q = A.D, the p x p Gram products
// fused into one reduction pass with fixed-order (deterministic, run-to-run
// reproducible) two-stage sums, Cholesky instead of LU for the step solves,
// beta's right-hand side formed algebraically as
//     R_new^T Q = R^T Q + alpha (Q^T Q)            (block_cg.hpp:262-264)
// and ONE fused pass for X += D alpha^T, R += Q alpha^T, D' = R + D beta^T
// (block_cg.hpp:222-244, :270-273).  Parity is "within tolerance" (X to 1e-8
// relative, pre-floor residual history), not bit-exact: DESIGN.md §2.
#pragma once
#include "common.cuh"

namespace coopcg_gpu {

constexpr int kFastBR = 64;   // rows per A panel (2 consumer warps x 32 rows)
constexpr int kFastT = 36;    // k per A tile; 36*8 B row stride keeps DMMA A-fragment loads conflict-free
constexpr int kFastS = 4;     // ring stages (two CTAs per SM; 5 stages at P = 8 measured slower:
                              // cfg 2 A.D 340 vs 314 us, cfg 1 unchanged -- round 2)
template <int P>
__host__ __device__ constexpr int fast_stages() { return kFastS; }

// Fast A layout ("tiles"): panel q (kFastBR rows), k-tile t: a contiguous
// [r][kk] block of kFastBR x kFastT doubles at ((q*ntiles + t)*BR + r)*T + kk.
// (index map: a_idx in common.cuh, ALay::fast)

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// (0) Operand re-layout for the MMA: a row-major n x P block (D or X) into
// k-tiles of [col][kk] (P x kFastT doubles per tile, zero past n), so the
// DMMA B-fragment loads (8 columns x 4 consecutive k per warp) hit distinct
// banks like the A fragments (288-byte stride) instead of 4-way conflicts.
template <int P>
__global__ void __launch_bounds__(256)
    operand_tiles_kernel(const double* __restrict__ src, int n, int ntiles, double* __restrict__ dst,
                         const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();  // after the wait: no chain of early launches reaches past this kernel
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    const size_t total = static_cast<size_t>(ntiles) * P * kFastT;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int kk = static_cast<int>(e % kFastT);
        const size_t rest = e / kFastT;
        const int col = static_cast<int>(rest % P);
        const int t = static_cast<int>(rest / P);
        const int k = t * kFastT + kk;
        dst[e] = (k < n) ? src[static_cast<size_t>(k) * P + col] : 0.0;
    }
}

// (1) Qpart[c] = A_panel(:, kchunk c) . D(kchunk c, :) for work units
// (panel, kchunk); persistent CTAs; warp 0 = bulk-copy producer, (8/MT)*WN
// warps consume with m8n8k4 DMMA: warp w covers 8*MT rows (MT M-tiles) x P/WN
// columns.  MT = 2 at P = 8: four consumer warps per CTA land on the four
// SM sub-partitions (a CTA's warps map to them by warp index), where two
// 32-row warps per CTA left the DMMA work of both co-resident CTAs on two
// of them (cfg 1: the busiest sub-partition's DMMA pipe ~80% active, round 2).  Both operands arrive as contiguous tiles (A: [r][kk], the
// operand: [col][kk]), one bulk copy each per stage.
// TR (transposed operand) = true: Dt holds [col][kk] k-tiles (P >= 16);
// false: Dt is the row-major n x P block itself (P = 8: its 64-byte rows
// already give conflict-free B fragments), tail rows zero-filled in smem.
template <int P, int WN, bool TR, int MT = 4>
__global__ void __launch_bounds__(32 + 32 * (kFastBR / (8 * MT)) * WN)
    ad_fast_kernel(const double* __restrict__ Af, int n, int n_loc, int ntiles, const double* __restrict__ Dt,
                   double* __restrict__ Qpart, int kchunks, int tiles_per_chunk, int nunits,
                   const int* __restrict__ stop, int res_t) {
    static_assert(P % (8 * WN) == 0, "fast contexts pad p to a multiple of 8 per column group");
    constexpr int NT = P / 8 / WN;  // N tiles of 8 columns per warp
    constexpr int NCW = (kFastBR / (8 * MT)) * WN;  // consumer warps
    constexpr int BR = kFastBR, T = kFastT, S = fast_stages<P>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);  // S x BR x T
    double* Ds = As + S * BR * T;                       // S x P x T
    uint64_t* full = reinterpret_cast<uint64_t*>(Ds + S * P * T);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        // Producer.  A does not change during a solve, so the first S A tiles
        // are requested BEFORE griddepcontrol.wait, while the previous kernel
        // (the iteration's tail, which triggers its dependents at its start)
        // is still running; the operand tiles (the previous kernel's output)
        // and everything after them follow the wait.  A stopped solve still
        // issues the operand copies of the prefetched stages and waits for
        // them, so no bulk copy is in flight when the CTA exits.
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy(), pol_res = l2_evict_last_policy();
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            bool waited = false;
            int pend_t[S];
            auto d_bytes = [&](int t) {
                return TR ? P * T * 8u : static_cast<uint32_t>(min(T, n - t * T)) * P * 8u;
            };
            // pdl_wait, then the operand copies of the prefetched stages;
            // false: the solve has stopped (the CTA drains and exits)
            auto release = [&](int npre) {
                pdl_wait();
                waited = true;
                for (int i = 0; i < npre; ++i)
                    bulk_g2s(Ds + i * P * T, Dt + static_cast<size_t>(pend_t[i]) * P * T, d_bytes(pend_t[i]), &full[i]);
                if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) {
                    for (int i = 0; i < npre; ++i) mbar_wait(&full[i], 0u);
                    return false;
                }
                return true;
            };
            // only the in-loop launches (stop != nullptr) prefetch: A is stable
            // across an iteration; setup / finalize / matvec_block launches may
            // follow a kernel that wrote A
            if (stop == nullptr) {
                pdl_wait();
                waited = true;
            }
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                const int q = u / kchunks, c = u % kchunks;
                const int t0 = c * tiles_per_chunk, t1 = min(ntiles, t0 + tiles_per_chunk);
                for (int t = t0; t < t1; ++t, ++it) {
                    if (it == S && !waited && !release(S)) return;
                    if (it >= S) mbar_wait(&empty[s], ph ^ 1u);
                    const uint32_t abytes = BR * T * 8u;
                    const uint32_t dbytes = d_bytes(t);
                    if (!TR) {  // row-major operand: copy the valid rows, zero the tail
                        const int rows = min(T, n - t * T);
                        double* ds = Ds + s * P * T;
                        for (int e = rows * P; e < T * P; ++e) ds[e] = 0.0;
                    }
                    mbar_arrive_expect_tx(&full[s], abytes + dbytes);
                    bulk_g2s_evict_first(As + s * BR * T, Af + (static_cast<size_t>(q) * ntiles + t) * BR * T, abytes, &full[s],
                                         (t - t0) < res_t ? pol_res : pol);
                    if (waited) bulk_g2s(Ds + s * P * T, Dt + static_cast<size_t>(t) * P * T, dbytes, &full[s]);
                    else pend_t[it] = t;
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            if (!waited) release(it);
        }
        return;
    }
    pdl_wait();
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    const int cw = warp - 1;
    const int rb = cw / WN;          // row block: rows [8 MT rb, 8 MT rb + 8 MT)
    const int cg = cw % WN;          // column group: N tiles [cg*NT, cg*NT + NT)
    const int g = lane >> 2, tg = lane & 3;
    int s = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int q = u / kchunks, c = u % kchunks;
        const int t0 = c * tiles_per_chunk, t1 = min(ntiles, t0 + tiles_per_chunk);
        double acc[MT][NT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        for (int t = t0; t < t1; ++t) {
            mbar_wait(&full[s], phase);
            const double* as = As + s * BR * T + (8 * MT * rb + g) * T + tg;
            // B fragment (k = tg, n = g): [col][kk] tiles read like A; row-major [kk][col] otherwise
            const double* ds = TR ? Ds + s * P * T + (8 * NT * cg + g) * T + tg
                                  : Ds + s * P * T + tg * P + 8 * NT * cg + g;
#pragma unroll
            for (int ks = 0; ks < T / 4; ++ks) {
                double a[MT], bb[NT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[mt] = as[8 * mt * T + 4 * ks];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bb[nt] = TR ? ds[8 * nt * T + 4 * ks] : ds[4 * ks * P + 8 * nt];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], bb[nt]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                phase ^= 1u;
            }
        }
        double* qp = Qpart + static_cast<size_t>(c) * n_loc * P;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int il = q * BR + 8 * MT * rb + 8 * mt + g;
            if (il < n_loc) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int col = 8 * (NT * cg + nt) + 2 * tg;
                    qp[static_cast<size_t>(il) * P + col] = acc[mt][nt][0];
                    qp[static_cast<size_t>(il) * P + col + 1] = acc[mt][nt][1];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// (2) Row pass after the MMA: dst = sum_c Qpart[c] (- b), written to the
// global rows row0.. of `dst`, plus per-CTA partial Grams over the rows:
//   mode 0 (iteration):  G0 = D^T Q, G1 = R^T D, G2 = R^T Q, G3 = Q^T Q
//   mode 1 (residual):   G0 = dst^T Q (if Q != null), diag(dst^T dst) -> G1[j][j]
// Rows are processed in tiles of 256/P (thread per element).
template <int P, bool PUSH = false>
__global__ void __launch_bounds__(256)
    // Qpart and dst may alias (kchunks == 1: the row pass rewrites the block it
    // sums in place), so neither is __restrict__.
    fast_rows_kernel(const double* Qpart, int kchunks, int n_loc, int row0, double* dst,
                     const double* __restrict__ b, const double* __restrict__ D, const double* __restrict__ R,
                     const double* __restrict__ Qfull, int p, int mode, double* __restrict__ partials,
                     const int* __restrict__ stop, PeerRows peers) {
    pdl_wait();
    if (stop != nullptr && *reinterpret_cast<volatile const int*>(stop)) return;
    constexpr int RP = 4;                 // rows per thread per tile (loads in flight together)
    constexpr int TR = (256 / P) * RP;    // rows per tile
    constexpr int NOUT = 4 * P * P;
    constexpr int PER = (NOUT + 255) / 256;
    __shared__ double tq[TR][P], td[TR][P], trr[TR][P];
    const int tid = threadIdx.x;
    const int lr0 = tid / P, j = tid % P;
    double acc[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) acc[q] = 0.0;
    const int ntile = (n_loc + TR - 1) / TR;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        double v[RP], dv[RP], rv[RP];
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int il = t * TR + lr0 + u * (256 / P);
            v[u] = 0.0;
            dv[u] = 0.0;
            rv[u] = 0.0;
            if (il < n_loc) {
                const int row = row0 + il;
                // k-chunk partial sums, chunks ascending; 8 loads in flight
                const double* qp = Qpart + static_cast<size_t>(il) * P + j;
                const size_t cs = static_cast<size_t>(n_loc) * P;
                for (int c0 = 0; c0 < kchunks; c0 += 8) {
                    double w[8];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) w[cc] = (c0 + cc < kchunks) ? qp[(c0 + cc) * cs] : 0.0;
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc)
                        if (c0 + cc < kchunks) v[u] += w[cc];
                }
                if (mode == 0) {
                    dv[u] = D[static_cast<size_t>(row) * P + j];
                    rv[u] = R[static_cast<size_t>(row) * P + j];
                } else if (Qfull != nullptr) {
                    dv[u] = Qfull[static_cast<size_t>(row) * P + j];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int lr = lr0 + u * (256 / P);
            const int il = t * TR + lr;
            if (il < n_loc) {
                const int row = row0 + il;
                if (b != nullptr) v[u] = (j < p) ? v[u] - b[row] : 0.0;
                const size_t o = static_cast<size_t>(row) * P + j;
                if (!PUSH) {
                    dst[o] = v[u];
                } else {
                    for (int q = 0; q < peers.n; ++q) peers.dst[q][o] = v[u];  // every rank's copy
                }
            }
            tq[lr][j] = v[u];
            td[lr][j] = dv[u];
            trr[lr][j] = rv[u];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int o = tid + q * 256;
            if (o < NOUT) {
                const int gsel = o / (P * P), a = (o / P) % P, c2 = o % P;
                // four independent accumulators over the tile rows (r mod 4),
                // added in a fixed order at the end of the tile
                const double(*xs)[P] = nullptr;
                const double(*ys)[P] = nullptr;
                if (mode == 0) {
                    xs = gsel == 0 ? td : (gsel == 3 ? tq : trr);
                    ys = (gsel == 1) ? td : tq;
                } else if (gsel == 0 && Qfull != nullptr) {
                    xs = tq;
                    ys = td;
                } else if (gsel == 1 && a == c2) {
                    xs = tq;
                    ys = tq;
                }
                if (xs != nullptr) {
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
                    for (int r = 0; r < TR; r += 4) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) s4[u] = fma(xs[r + u][a], ys[r + u][c2], s4[u]);
                    }
                    acc[q] += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int o = tid + q * 256;
        if (o < NOUT) partials[static_cast<size_t>(blockIdx.x) * NOUT + o] = acc[q];
    }
    if (PUSH) __threadfence_system();
}

// ---------------------------------------------------------------------------
// (3) Step matrices on one CTA: reduce the Gram partials, then warp 0 runs
// the SPD guard (block_cg.hpp:196-202), Cholesky of M = sym(D^T Q) with the
// reference's pivot floor max|M| * 1e-14 (block_cg.hpp:180-190), and solves
//   alpha_i: M alpha_i^T = -(R^T D)_i            (block_cg.hpp:203-217)
//   beta_i:  M beta_i^T  = -(R^T Q + alpha Q^T Q)_i   (algebraic R_new^T Q)
// mode 0: alpha + beta; mode 1: alpha only (recompute iteration, beta later);
// mode 2: beta only from G0 = R_new^T Q of a residual pass (uses ctl->lu).
// L L^T x = rhs for lane-owned right-hand sides, L in shared memory with
// 1 / L_ii stored on its diagonal (no division on the solve's critical path).
#ifndef COOPCG_CTA_SOLVE_MIN_P
#define COOPCG_CTA_SOLVE_MIN_P 16
#endif
// The step solves on a whole CTA in shared memory (P >= COOPCG_CTA_SOLVE_MIN_P, where one warp
// holding P-wide register rows spills and serialises: 27 us at P = 16 in the
// fused kernel, 394 us at P = 32 in fast_solve_kernel, round 2).
//   M = sym(G0) (identity on the padded rows), SPD guard, right-looking
//   Cholesky by warp 0 (lane = row; the factor keeps 1 / L_kk on its
//   diagonal, the format of ctl->lu), W = L^-1 column by column, Minv = W^T W,
//   then alpha_i = Minv (-G1_i), rhs_beta = -(G2 + alpha G3), beta_i = Minv rhs_i
//   as CTA-wide products.  mode 0: alpha + beta; 1: alpha; 2: beta from the
//   stored factor `lf` (filled by the caller) with rhs -G0.
// Returns 0, 1 (pivot vanished: rank collapse) or 2 (SPD guard); every
// thread of the CTA must call it.  Shared buffers: lf, W, Mi, al, be (P x P+1).
template <int P>
__device__ int solve_cta(const double* G, int p, int mode, const double* __restrict__ nsq,
                         double (*lf)[P + 1], double (*W)[P + 1], double (*Mi)[P + 1], double (*al)[P + 1],
                         double (*be)[P + 1], double* red) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int flag;
    auto g = [&](int gsel, int a, int c) { return G[(gsel * P + a) * P + c]; };
    if (mode != 2) {
        double mx = 0.0;
        for (int e = tid; e < P * P; e += nt) {
            const int i = e / P, j = e % P;
            double v = (i == j) ? 1.0 : 0.0;
            if (i < p && j < p) {
                v = 0.5 * (g(0, i, j) + g(0, j, i));
                mx = fmax(mx, fabs(v));
            }
            lf[i][j] = v;
        }
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0) red[warp] = mx;
        if (tid == 0) flag = 0;
        __syncthreads();
        if (tid < p && !(lf[tid][tid] > 0.0) && nsq[tid] > 0.0) atomicOr(&flag, 2);  // block_cg.hpp:196-202
        if (warp == 0) {
            double m2 = (lane < nt / 32) ? red[lane] : 0.0;
            for (int off = 16; off > 0; off >>= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, off));
            const double floor = m2 * 1e-14;  // the reference's pivot floor (block_cg.hpp:180-190)
            __syncwarp();
            if (flag == 0) {
                for (int k = 0; k < p; ++k) {
                    const double d = lf[k][k];
                    if (!(d > floor)) {
                        if (lane == 0) flag = 1;
                        break;
                    }
                    const double inv = rsqrt(d);
                    if (lane > k && lane < p) lf[lane][k] *= inv;
                    __syncwarp();
                    if (lane > k && lane < p) {
                        const double lik = lf[lane][k];
                        for (int j = k + 1; j <= lane; ++j) lf[lane][j] = fma(-lik, lf[j][k], lf[lane][j]);
                    }
                    if (lane == k) lf[k][k] = inv;
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        if (flag) return flag;
    }
    // W = L^-1 (lower), one column per thread of warp 0
    if (warp == 0) {
        const int j = lane;
        for (int i = 0; i < P; ++i) {
            double w = 0.0;
            if (j < p && i < p && i >= j) {
                double s = (i == j) ? 1.0 : 0.0;
                for (int m = j; m < i; ++m) s = fma(-lf[i][m], W[m][j], s);
                w = s * lf[i][i];
            }
            if (j < P) W[i][j] = w;
            __syncwarp();
        }
    }
    __syncthreads();
    // Minv = W^T W
    for (int e = tid; e < P * P; e += nt) {
        const int a = e / P, b = e % P;
        double s = 0.0;
        if (a < p && b < p)
            for (int m = (a > b ? a : b); m < p; ++m) s = fma(W[m][a], W[m][b], s);
        Mi[a][b] = s;
    }
    __syncthreads();
    if (mode != 2) {
        // alpha_i = Minv (-G1_i)   (block_cg.hpp:203-217)
        for (int e = tid; e < P * P; e += nt) {
            const int i = e / P, j = e % P;
            double s = 0.0;
            if (i < p && j < p)
                for (int m = 0; m < p; ++m) s = fma(Mi[j][m], -g(1, i, m), s);
            al[i][j] = s;
        }
        __syncthreads();
    }
    if (mode == 1) return 0;
    // rhs_beta (W reused): -(G2 + alpha G3), or -G0 from a residual pass (mode 2)
    for (int e = tid; e < P * P; e += nt) {
        const int i = e / P, j = e % P;
        double s = 0.0;
        if (i < p && j < p) {
            if (mode == 2) {
                s = -g(0, i, j);
            } else {
                s = g(2, i, j);
                for (int m = 0; m < p; ++m) s = fma(al[i][m], g(3, m, j), s);
                s = -s;
            }
        }
        W[i][j] = s;
    }
    __syncthreads();
    for (int e = tid; e < P * P; e += nt) {
        const int i = e / P, j = e % P;
        double s = 0.0;
        if (i < p && j < p)
            for (int m = 0; m < p; ++m) s = fma(Mi[j][m], W[i][m], s);
        be[i][j] = s;
    }
    __syncthreads();
    return 0;
}

template <int P>
__device__ __forceinline__ void chol_solve_regs(const double (*l)[P + 1], int p, const double (&rhs)[P],
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
            double s = rhs[i];
#pragma unroll
            for (int j = 0; j < i; ++j) s = fma(-l[i][j], y[j], s);
            y[i] = s * l[i][i];  // the diagonal holds 1 / L_ii
        }
    }
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
        if (i < p) {
            double s = y[i];
#pragma unroll
            for (int j = i + 1; j < P; ++j)
                if (j < p) s = fma(-l[j][i], x[j], s);
            x[i] = s * l[i][i];
        }
    }
}

template <int P>
__global__ void __launch_bounds__(1024)
    fast_solve_kernel(const double* __restrict__ partials, int nparts, double* __restrict__ small, Ctl* ctl,
                      int mode) {
    pdl_wait();
    if (*reinterpret_cast<volatile int*>(&ctl->stop)) return;
    extern __shared__ __align__(16) double dyn[];  // flat[4 P P] then red[blockDim]
    double* flat = dyn;
    double* red = dyn + 4 * P * P;
    __shared__ double lsm[P][P + 1];
    const int p = ctl->p;
    const SmallLayout L{P};
    const int tid = threadIdx.x;
    const int nout = (mode == 2) ? P * P : 4 * P * P;
    // inputs of warp 0 requested before the reduction
    double nsq = 0.0, lu_in[P];
    if (tid < P) {
        nsq = small[L.nsq_d() + tid];
#pragma unroll
        for (int j = 0; j < P; ++j) lu_in[j] = (mode == 2) ? ctl->lu[tid * P + j] : 0.0;
    }
    cta_reduce_fixed(partials, nparts, 4 * P * P, 0, 1, nout, flat, red);
    __syncthreads();
    if constexpr (P >= COOPCG_CTA_SOLVE_MIN_P) {
        // the whole CTA solves in shared memory (solve_cta); buffers after red[]
        double(*lf)[P + 1] = reinterpret_cast<double(*)[P + 1]>(red + blockDim.x);
        double(*Wb)[P + 1] = lf + P;
        double(*Mib)[P + 1] = lf + 2 * P;
        double(*al)[P + 1] = lf + 3 * P;
        double(*be)[P + 1] = lf + 4 * P;
        if (mode == 2) {
            for (int e = tid; e < P * P; e += blockDim.x) lf[e / P][e % P] = ctl->lu[e];
            __syncthreads();
        }
        const int rc = solve_cta<P>(flat, p, mode, small + L.nsq_d(), lf, Wb, Mib, al, be, red);
        if (rc) {
            if (tid == 0) {
                if (rc == 2) {
                    ctl->err = 2;
                    ctl->err_iter = ctl->k;
                } else {
                    ctl->status = 1;  // rank collapse (pivot vanished)
                }
                ctl->stop = 1;
            }
            return;
        }
        for (int e = tid; e < P * P; e += blockDim.x) {
            const int i = e / P, j = e % P;
            if (mode != 2) {
                ctl->lu[e] = lf[i][j];
                small[L.alpha() + e] = al[i][j];
            }
            if (mode != 1) small[L.beta() + e] = be[i][j];
        }
        return;
    }
    // G[gsel][a][c] = flat[(gsel * P + a) * P + c]
    auto G = [&](int gsel, int a, int c) { return flat[(gsel * P + a) * P + c]; };
    if (tid >= 32) return;
    const int lane = tid;
    double x[P], rhs[P];
    if (mode != 2) {
        // M = (raw + raw^T)/2, floor = max|M| * 1e-14; lane i holds row i
        double l[P];
        double maxabs = 0.0, diag = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            l[j] = 0.0;
            if (lane < p && j < p) {
                l[j] = 0.5 * (G(0, lane, j) + G(0, j, lane));
                maxabs = fmax(maxabs, fabs(l[j]));
                if (j == lane) diag = l[j];
            }
        }
        for (int off = 16; off > 0; off >>= 1) maxabs = fmax(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, off));
        const double floor = maxabs * 1e-14;
        const bool bad = (lane < p) && !(diag > 0.0) && (nsq > 0.0);
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) {
                ctl->err = 2;
                ctl->err_iter = ctl->k;
                ctl->stop = 1;
            }
            return;
        }
        // Cholesky (lower, left-looking; lane owns row; row k broadcast by shuffle)
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (k >= p) break;
            double dk = 0.0;
            if (lane == k) {
                double s = l[k];
#pragma unroll
                for (int m = 0; m < k; ++m) s = fma(-l[m], l[m], s);
                dk = (s > floor) ? rsqrt(s) : -1.0;  // 1 / L_kk
            }
            const double ikk = __shfl_sync(0xffffffffu, dk, k);
            if (!(ikk > 0.0)) {
                if (lane == 0) {
                    ctl->status = 1;  // rank collapse (pivot vanished)
                    ctl->stop = 1;
                }
                return;
            }
            double rk[P];
#pragma unroll
            for (int m = 0; m < k; ++m) rk[m] = __shfl_sync(0xffffffffu, l[m], k);
            if (lane > k && lane < p) {
                double s = l[k];
#pragma unroll
                for (int m = 0; m < k; ++m) s = fma(-l[m], rk[m], s);
                l[k] = s * ikk;
            }
            if (lane == k) l[k] = ikk;  // the factor keeps 1 / L_kk on its diagonal
        }
        if (lane < P) {
#pragma unroll
            for (int j = 0; j < P; ++j) {
                lsm[lane][j] = l[j];
                ctl->lu[lane * P + j] = l[j];
            }
        }
        __syncwarp();
        if (lane < p) {
#pragma unroll
            for (int j = 0; j < P; ++j) rhs[j] = (j < p) ? -G(1, lane, j) : 0.0;
            chol_solve_regs<P>(lsm, p, rhs, x);
#pragma unroll
            for (int j = 0; j < P; ++j) small[L.alpha() + lane * P + j] = (j < p) ? x[j] : 0.0;
            if (mode == 0) {
                // rhs_beta(i, j) = -(R^T Q + alpha Q^T Q)(i, j)
#pragma unroll
                for (int j = 0; j < P; ++j) {
                    double s = G(2, lane, j);
#pragma unroll
                    for (int m = 0; m < P; ++m)
                        if (m < p) s = fma(x[m], G(3, m, j), s);
                    rhs[j] = (j < p) ? -s : 0.0;
                }
                double xb[P];
                chol_solve_regs<P>(lsm, p, rhs, xb);
#pragma unroll
                for (int j = 0; j < P; ++j) small[L.beta() + lane * P + j] = (j < p) ? xb[j] : 0.0;
            }
        }
    } else {
        if (lane < P) {
#pragma unroll
            for (int j = 0; j < P; ++j) lsm[lane][j] = lu_in[j];
        }
        __syncwarp();
        if (lane < p) {
#pragma unroll
            for (int j = 0; j < P; ++j) rhs[j] = (j < p) ? -G(0, lane, j) : 0.0;
            chol_solve_regs<P>(lsm, p, rhs, x);
#pragma unroll
            for (int j = 0; j < P; ++j) small[L.beta() + lane * P + j] = (j < p) ? x[j] : 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// (4) The fused update pass (one read of X, R, D, Q; one write of X, R, D'):
//   mode 0: X += D alpha^T; R += Q alpha^T; D' = R + D beta^T
//   mode 1: X += D alpha^T only (recompute iteration)
//   mode 2: D' = R + D beta^T only (after the recompute)
// plus per-CTA partials of |R_j|^2 (P values; modes 0) and the pairs of
// D'^T D' (rank certificate, the exact path's beta_direction_kernel format).
template <int P>
__global__ void __launch_bounds__(256)
    fast_update_kernel(double* __restrict__ X, double* __restrict__ R, const double* __restrict__ Q,
                       const double* __restrict__ D, double* __restrict__ Dn, const double* __restrict__ small, int n,
                       int p, int mode, double* __restrict__ norm_part, double* __restrict__ pair_part,
                       const int* __restrict__ stop) {
    pdl_wait();
    pdl_trigger();  // after the wait: no chain of early launches reaches past this kernel
    if (*reinterpret_cast<volatile const int*>(stop)) return;
    constexpr int RP = (P >= 32) ? 2 : 4;
    constexpr int TR = (256 / P) * RP;
    const SmallLayout L{P};
    __shared__ double al[P][P + 1], be[P][P + 1];
    __shared__ double tr_[TR][P], tdn[TR][P], td_[TR][P], tq_[TR][P];
    const int tid = threadIdx.x;
    for (int idx = tid; idx < p * p; idx += 256) {
        al[idx / p][idx % p] = small[L.alpha() + (idx / p) * P + idx % p];
        be[idx / p][idx % p] = small[L.beta() + (idx / p) * P + idx % p];
    }
    // D'^T D' pair partials: item (pair, g) sums the tile rows r = g, g + G, ...
    // (G = 256 / npairs row groups per pair when the pairs are fewer than the
    // threads), so no thread walks a whole tile in one dependent chain; the G
    // group sums are added in a fixed order at the end (deterministic).
    const int npairs = p * (p + 1) / 2;
    const int G = npairs < 256 ? 256 / npairs : 1;
    int pi[3], pj[3], pg[3];
    double part[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        int t = tid + q * 256;
        pi[q] = pj[q] = -1;
        pg[q] = 0;
        if (t < npairs * G) {
            pg[q] = t % G;
            t /= G;
            int i = 0;
            while (t >= p - i) {
                t -= p - i;
                ++i;
            }
            pi[q] = i;
            pj[q] = i + t;
        }
    }
    double nrm = 0.0;
    const int lr0 = tid / P, i = tid % P;
    __syncthreads();
    const int ntile = (n + TR - 1) / TR;
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        // stage the D (and Q) rows of the tile: loads for RP rows in flight together
        double dv[RP], qv[RP], xv[RP], rv[RP];
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int row = t * TR + lr0 + u * (256 / P);
            const size_t e = static_cast<size_t>(row) * P + i;
            const bool ok = row < n;
            dv[u] = ok ? D[e] : 0.0;
            qv[u] = (ok && mode == 0) ? Q[e] : 0.0;
            xv[u] = (ok && mode <= 1) ? X[e] : 0.0;
            rv[u] = (ok && mode != 1) ? R[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            td_[lr0 + u * (256 / P)][i] = dv[u];
            tq_[lr0 + u * (256 / P)][i] = qv[u];
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int lr = lr0 + u * (256 / P);
            const int row = t * TR + lr;
            const size_t e = static_cast<size_t>(row) * P + i;
            double rnew = 0.0;
            if (row < n && i < p) {
                if (mode <= 1) {
                    double x = xv[u];
                    for (int j = 0; j < p; ++j) x = fma(al[i][j], td_[lr][j], x);
                    X[e] = x;
                }
                if (mode == 0) {
                    double r = rv[u];
                    for (int j = 0; j < p; ++j) r = fma(al[i][j], tq_[lr][j], r);
                    R[e] = r;
                    rnew = r;
                    nrm = fma(r, r, nrm);
                } else {
                    rnew = rv[u];
                }
            }
            tr_[lr][i] = rnew;
        }
        __syncthreads();
        if (mode != 1) {
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int lr = lr0 + u * (256 / P);
                const int row = t * TR + lr;
                double dn = 0.0;
                if (row < n && i < p) {
                    dn = tr_[lr][i];
                    for (int j = 0; j < p; ++j) dn = fma(be[i][j], td_[lr][j], dn);
                }
                if (row < n) Dn[static_cast<size_t>(row) * P + i] = dn;
                tdn[lr][i] = dn;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (pi[q] >= 0) {
                    double s = part[q];
                    for (int r = pg[q]; r < TR; r += G) s = fma(tdn[r][pi[q]], tdn[r][pj[q]], s);
                    part[q] = s;
                }
        }
        __syncthreads();
    }
    // column norms: threads with the same i (tid % P) hold partial sums; reduce
    // them in a fixed order through shared memory.
    __shared__ double nred[256];
    nred[tid] = nrm;
    __syncthreads();
    if (tid < P) {
        double s = 0.0;
        for (int r = 0; r < 256 / P; ++r) s += nred[r * P + tid];
        if (mode == 0) norm_part[static_cast<size_t>(blockIdx.x) * P + tid] = s;
    }
    if (mode != 1) {
        if (G == 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (pi[q] >= 0) pair_part[static_cast<size_t>(blockIdx.x) * npairs + tid + q * 256] = part[q];
        } else {  // one item per thread: add the G group sums of each pair in order
            __syncthreads();
            nred[tid] = part[0];
            __syncthreads();
            if (tid < npairs) {
                double t = 0.0;
                for (int g = 0; g < G; ++g) t += nred[tid * G + g];
                pair_part[static_cast<size_t>(blockIdx.x) * npairs + tid] = t;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// (4b) One fused, cooperative launch for the whole post-MMA part of a plain
// (non-recompute, single-GPU) iteration: the row pass, the Gram reduction,
// the step solves and the update pass of kernels (2)-(4), separated by two
// grid-wide barriers (every CTA is co-resident: cooperative launch).
//   A  rows:   Q = sum_c Qpart[c]; per-CTA partials of D^T Q, R^T D, R^T Q, Q^T Q
//   B  reduce: one warp per Gram entry sums the CTA partials (fixed order)
//   C  solve:  every CTA redoes the Cholesky / alpha / beta solve from the
//              reduced Grams in shared memory (identical inputs -> identical
//              results); CTA 0 publishes alpha, beta, the factor and errors
//   D  update: X += D alpha^T, R += Q alpha^T, D' = R + D beta^T, plus the
//              |R_j|^2 and D'^T D' per-CTA partials (kernel (4)'s format)
// Three launches and their drain/fill gaps become one.  The per-element
// arithmetic is that of the separate kernels; only the Gram reduction adds
// the CTA partials in a different (still fixed, deterministic) order.
// COOPCG_PHASE_TIMES (measurement builds only, tools/variants.sh): CTA 0's
// thread 0 accumulates the globaltimer time of each phase of fast_iter_kernel
// into g_phase_ns[0..6] (entry->A end, barrier 1, B, barrier 2, C loads,
// C solve + sync, D), g_phase_ns[7] = launches; printed at context destroy.
#ifdef COOPCG_PHASE_TIMES
__device__ unsigned long long g_phase_ns[16];
#define PHASE_MARK(i)                                                                  \
    do {                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                     \
            const unsigned long long now_ = globaltimer_ns();                          \
            if ((i) > 0) atomicAdd(&g_phase_ns[(i) > 7 ? (i) : (i) - 1], now_ - t_prev_);\
            t_prev_ = now_;                                                            \
        }                                                                              \
    } while (0)
#define PHASE_SUB(i)                                                                   \
    do {                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                     \
            const unsigned long long now_ = globaltimer_ns();                          \
            atomicAdd(&g_phase_ns[i], now_ - t_sub_);                                  \
            t_sub_ = now_;                                                             \
        }                                                                              \
    } while (0)
#else
#define PHASE_SUB(i) \
    do {             \
    } while (0)
#define PHASE_MARK(i) \
    do {              \
    } while (0)
#endif
// Grid barrier on a monotonic 64-bit arrival counter (never reset): CTA
// arrival j of a barrier round returns old = r * G + j, so the round ends
// when the counter reaches (r + 1) * G.  One release atomic per CTA, then
// acquire polls; no reset atomics on the last arriver's critical path.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long old;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        const unsigned long long target = (old / nblocks + 1) * nblocks;
        unsigned long long cur;
        do {
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(bar) : "memory");
        } while (cur < target);
    }
    __syncthreads();
}

template <int P, int RP>
__host__ __device__ constexpr int fused_rows_tr() { return (256 / P) * RP; }
template <int P, int RP>
__host__ __device__ constexpr int fused_upd_tr() { return (256 / P) * RP; }
template <int P, int RP>
__host__ __device__ constexpr size_t fused_smem_bytes() {
    // phase A's three tiles (kept for phase D when the tilings agree), then phase
    // C/D: grams (4 P^2) + alpha, beta + 4 update tiles + reductions + the factor
    constexpr size_t a = 3ull * fused_rows_tr<P, RP>() * P;
    constexpr size_t d = 4ull * P * P + 2ull * P * (P + 1) + 4ull * fused_upd_tr<P, RP>() * P + 256 + P * (P + 1);
    constexpr size_t e = P >= COOPCG_CTA_SOLVE_MIN_P ? 2ull * P * (P + 1) : 0;  // solve_cta's W and Minv
    return (a + d + e) * sizeof(double);
}

template <int P, int RP>
__global__ void __launch_bounds__(256, 2)
    fast_iter_kernel(const double* __restrict__ Qpart, int kchunks, int n, double* __restrict__ Q,
                     double* __restrict__ X, double* __restrict__ R, const double* __restrict__ D,
                     double* __restrict__ Dn, double* __restrict__ small, Ctl* ctl, int p,
                     double* __restrict__ gpart, double* __restrict__ gfin, double* __restrict__ norm_part,
                     double* __restrict__ pair_part, unsigned long long* __restrict__ gbar) {
    pdl_wait();
    pdl_trigger();  // after the wait: no chain of early launches reaches past this kernel
    if (*reinterpret_cast<volatile const int*>(&ctl->stop)) return;  // stable: no writer runs concurrently
    unsigned long long t_prev_ = 0, t_sub_ = 0;
    (void)t_prev_;
    (void)t_sub_;
    PHASE_MARK(0);
    extern __shared__ __align__(16) double fsm[];
    constexpr int NOUT = 4 * P * P;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned int G = gridDim.x;
    const SmallLayout L{P};

    // When the row pass and the update pass tile the rows alike and every CTA
    // owns at most one tile, the update reuses the row pass's D, Q, R tiles
    // (still in shared memory) and X is fetched during the row pass.
    constexpr int TRA = fused_rows_tr<P, RP>();
    constexpr bool SAME_TILING = TRA == fused_upd_tr<P, RP>();
    const bool reuse = SAME_TILING && (n + TRA - 1) / TRA <= static_cast<int>(gridDim.x);
    double xpre[RP];
#pragma unroll
    for (int u = 0; u < RP; ++u) xpre[u] = 0.0;
    // ---- A: row pass (kernel (2), mode 0) ----------------------------------
    {
        constexpr int TR = TRA;
        constexpr int PER = (NOUT + 255) / 256;
        double(*tq)[P] = reinterpret_cast<double(*)[P]>(fsm);
        double(*td)[P] = reinterpret_cast<double(*)[P]>(fsm + TR * P);
        double(*trr)[P] = reinterpret_cast<double(*)[P]>(fsm + 2 * TR * P);
        const int lr0 = tid / P, j = tid % P;
        if (reuse) {
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int il = blockIdx.x * TR + lr0 + u * (256 / P);
                if (il < n) xpre[u] = X[static_cast<size_t>(il) * P + j];
            }
        }
        double acc[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) acc[q] = 0.0;
        const int ntile = (n + TR - 1) / TR;
        for (int t = blockIdx.x; t < ntile; t += G) {
            double v[RP], dv[RP], rv[RP];
            const size_t cs = static_cast<size_t>(n) * P;
            if (kchunks <= 8) {
                // every row's chunk partials in flight together, then summed in chunk order
                double w[RP][8];
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    const int il = t * TR + lr0 + u * (256 / P);
                    const double* qp = Qpart + static_cast<size_t>(il) * P + j;
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) w[u][cc] = (il < n && cc < kchunks) ? qp[cc * cs] : 0.0;
                    dv[u] = (il < n) ? D[static_cast<size_t>(il) * P + j] : 0.0;
                    rv[u] = (il < n) ? R[static_cast<size_t>(il) * P + j] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    v[u] = 0.0;
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc)
                        if (cc < kchunks) v[u] += w[u][cc];
                }
            } else {
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    const int il = t * TR + lr0 + u * (256 / P);
                    v[u] = dv[u] = rv[u] = 0.0;
                    if (il < n) {
                        const double* qp = Qpart + static_cast<size_t>(il) * P + j;
                        for (int c0 = 0; c0 < kchunks; c0 += 8) {
                            double w[8];
#pragma unroll
                            for (int cc = 0; cc < 8; ++cc) w[cc] = (c0 + cc < kchunks) ? qp[(c0 + cc) * cs] : 0.0;
#pragma unroll
                            for (int cc = 0; cc < 8; ++cc)
                                if (c0 + cc < kchunks) v[u] += w[cc];
                        }
                        dv[u] = D[static_cast<size_t>(il) * P + j];
                        rv[u] = R[static_cast<size_t>(il) * P + j];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int lr = lr0 + u * (256 / P);
                const int il = t * TR + lr;
                if (il < n) Q[static_cast<size_t>(il) * P + j] = v[u];
                tq[lr][j] = v[u];
                td[lr][j] = dv[u];
                trr[lr][j] = rv[u];
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int o = tid + q * 256;
                if (o < NOUT) {
                    const int gsel = o / (P * P), a = (o / P) % P, c2 = o % P;
                    const double(*xs)[P] = gsel == 0 ? td : (gsel == 3 ? tq : trr);
                    const double(*ys)[P] = (gsel == 1) ? td : tq;
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 2
                    for (int r = 0; r < TR; r += 4) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) s4[u] = fma(xs[r + u][a], ys[r + u][c2], s4[u]);
                    }
                    acc[q] += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int o = tid + q * 256;
            if (o < NOUT) gpart[static_cast<size_t>(blockIdx.x) * NOUT + o] = acc[q];
        }
    }
    PHASE_MARK(1);
    grid_barrier(gbar, G);
    PHASE_MARK(2);

    // ---- B: Gram reduction, one warp per entry (fixed order) ---------------
    for (int o = blockIdx.x * 8 + warp; o < NOUT; o += G * 8) {
        // lane l sums partials l, l+32, ... (G <= 296: at most 10), loads first
        double v[10];
#pragma unroll
        for (int q = 0; q < 10; ++q) {
            const unsigned int c = lane + 32u * q;
            v[q] = (c < G) ? __ldcg(gpart + static_cast<size_t>(c) * NOUT + o) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 10; ++q) s += v[q];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) gfin[o] = s;
    }
    PHASE_MARK(3);
    grid_barrier(gbar, G);
    PHASE_MARK(4);

    // ---- C: step solves (kernel (3), mode 0), redundantly in every CTA ------
    double* flat = fsm + 3 * TRA * P;            // 4 P^2 (after phase A's tiles)
    double(*al)[P + 1] = reinterpret_cast<double(*)[P + 1]>(flat + NOUT);
    double(*be)[P + 1] = reinterpret_cast<double(*)[P + 1]>(flat + NOUT + P * (P + 1));
    double* tiles = flat + NOUT + 2 * P * (P + 1);
    constexpr int TRU = fused_upd_tr<P, RP>();
    double* nred = tiles + 4 * TRU * P;          // 256
    double(*lsm)[P + 1] = reinterpret_cast<double(*)[P + 1]>(nred + 256);
    __shared__ int abort_flag;
    for (int o = tid; o < NOUT; o += 256) flat[o] = __ldcg(gfin + o);
    if (tid == 0) abort_flag = 0;
    __syncthreads();
    PHASE_MARK(5);
#ifdef COOPCG_PHASE_TIMES
    if (blockIdx.x == 0 && threadIdx.x == 0) t_sub_ = t_prev_;
#endif
    auto Gm = [&](int gsel, int a, int c) { return flat[(gsel * P + a) * P + c]; };
    if constexpr (P >= COOPCG_CTA_SOLVE_MIN_P) {
        double(*Wb)[P + 1] = reinterpret_cast<double(*)[P + 1]>(&lsm[P][0]);
        double(*Mib)[P + 1] = reinterpret_cast<double(*)[P + 1]>(&lsm[2 * P][0]);
        const int rc = solve_cta<P>(flat, p, 0, small + L.nsq_d(), lsm, Wb, Mib, al, be, nred);
        if (rc) {
            if (blockIdx.x == 0 && tid == 0) {
                if (rc == 2) {
                    ctl->err = 2;
                    ctl->err_iter = ctl->k;
                } else {
                    ctl->status = 1;  // rank collapse (pivot vanished)
                }
                ctl->stop = 1;
            }
            return;
        }
        if (blockIdx.x == 0)
            for (int e = tid; e < P * P; e += 256) {
                const int i = e / P, j = e % P;
                ctl->lu[e] = lsm[i][j];
                small[L.alpha() + e] = al[i][j];
                small[L.beta() + e] = be[i][j];
            }
    } else {
        // The solve runs on one warp; the two CTAs an SM hosts (blocks b and
        // b + #SMs under the usual placement) use warps 0 and 1, i.e. different
        // SMSPs, so their serial FP64 chains do not share an issue port.
        unsigned int nsm;
        asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
        const int solver = static_cast<int>((blockIdx.x / nsm) & 1u);
        if (warp == solver) {
            const bool pub = blockIdx.x == 0;
            const double nsq = (lane < P) ? small[L.nsq_d() + lane] : 0.0;
            double l[P];
            double maxabs = 0.0, diag = 0.0;
#pragma unroll
            for (int jj = 0; jj < P; ++jj) {
                l[jj] = 0.0;
                if (lane < p && jj < p) {
                    l[jj] = 0.5 * (Gm(0, lane, jj) + Gm(0, jj, lane));
                    maxabs = fmax(maxabs, fabs(l[jj]));
                    if (jj == lane) diag = l[jj];
                }
            }
            for (int off = 16; off > 0; off >>= 1) maxabs = fmax(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, off));
            const double floor = maxabs * 1e-14;
            PHASE_SUB(8);
            const bool bad = (lane < p) && !(diag > 0.0) && (nsq > 0.0);
            bool fail = false;
            if (__any_sync(0xffffffffu, bad)) {
                if (pub && lane == 0) {
                    ctl->err = 2;
                    ctl->err_iter = ctl->k;
                    ctl->stop = 1;
                }
                fail = true;
            }
#pragma unroll
            for (int k = 0; k < P; ++k) {
                if (fail || k >= p) break;
                double dk = 0.0;
                if (lane == k) {
                    double sk = l[k];
#pragma unroll
                    for (int m = 0; m < k; ++m) sk = fma(-l[m], l[m], sk);
                    dk = (sk > floor) ? rsqrt(sk) : -1.0;  // 1 / L_kk
                }
                const double ikk = __shfl_sync(0xffffffffu, dk, k);
                if (!(ikk > 0.0)) {
                    if (pub && lane == 0) {
                        ctl->status = 1;  // rank collapse (pivot vanished)
                        ctl->stop = 1;
                    }
                    fail = true;
                    break;
                }
                double rk[P];
#pragma unroll
                for (int m = 0; m < k; ++m) rk[m] = __shfl_sync(0xffffffffu, l[m], k);
                if (lane > k && lane < p) {
                    double sk = l[k];
#pragma unroll
                    for (int m = 0; m < k; ++m) sk = fma(-l[m], rk[m], sk);
                    l[k] = sk * ikk;
                }
                if (lane == k) l[k] = ikk;  // 1 / L_kk on the diagonal
            }
            PHASE_SUB(9);
            if (fail) {
                if (lane == 0) abort_flag = 1;
            } else {
                if (lane < P) {
#pragma unroll
                    for (int jj = 0; jj < P; ++jj) {
                        lsm[lane][jj] = l[jj];
                        if (pub) ctl->lu[lane * P + jj] = l[jj];
                    }
                }
                __syncwarp();
                double x[P], rhs[P], xb[P];
                if (lane < p) {
#pragma unroll
                    for (int jj = 0; jj < P; ++jj) rhs[jj] = (jj < p) ? -Gm(1, lane, jj) : 0.0;
                    chol_solve_regs<P>(lsm, p, rhs, x);
                    PHASE_SUB(10);
#pragma unroll
                    for (int jj = 0; jj < P; ++jj) {
                        double sb = Gm(2, lane, jj);
#pragma unroll
                        for (int m = 0; m < P; ++m)
                            if (m < p) sb = fma(x[m], Gm(3, m, jj), sb);
                        rhs[jj] = (jj < p) ? -sb : 0.0;
                    }
                    chol_solve_regs<P>(lsm, p, rhs, xb);
                    PHASE_SUB(11);
#pragma unroll
                    for (int jj = 0; jj < P; ++jj) {
                        al[lane][jj] = (jj < p) ? x[jj] : 0.0;
                        be[lane][jj] = (jj < p) ? xb[jj] : 0.0;
                        if (pub) {
                            small[L.alpha() + lane * P + jj] = (jj < p) ? x[jj] : 0.0;
                            small[L.beta() + lane * P + jj] = (jj < p) ? xb[jj] : 0.0;
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    PHASE_MARK(6);
    if (abort_flag) return;

    // ---- D: update pass (kernel (4), mode 0) -------------------------------
    {
        constexpr int TR = TRU;
        double(*tr_)[P] = reinterpret_cast<double(*)[P]>(tiles);
        double(*tdn)[P] = reinterpret_cast<double(*)[P]>(tiles + TR * P);
        // with `reuse`, D and Q are phase A's tiles (tq at fsm, td after it)
        double(*td_)[P] = reinterpret_cast<double(*)[P]>(reuse ? fsm + TRA * P : tiles + 2 * TR * P);
        double(*tq_)[P] = reinterpret_cast<double(*)[P]>(reuse ? fsm : tiles + 3 * TR * P);
        const double(*trA)[P] = reinterpret_cast<const double(*)[P]>(fsm + 2 * TRA * P);
        const int npairs = p * (p + 1) / 2;
        const int GR = npairs < 256 ? 256 / npairs : 1;
        int pi[3], pj[3], pg[3];
        double part[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            int t = tid + q * 256;
            pi[q] = pj[q] = -1;
            pg[q] = 0;
            if (t < npairs * GR) {
                pg[q] = t % GR;
                t /= GR;
                int i = 0;
                while (t >= p - i) {
                    t -= p - i;
                    ++i;
                }
                pi[q] = i;
                pj[q] = i + t;
            }
        }
        double nrm = 0.0;
        const int lr0 = tid / P, i = tid % P;
        const int ntile = (n + TR - 1) / TR;
        for (int t = blockIdx.x; t < ntile; t += G) {
            double dv[RP], qv[RP], xv[RP], rv[RP];
            if (reuse) {  // one tile per CTA: the row pass's tiles and the prefetched X
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    xv[u] = xpre[u];
                    rv[u] = trA[lr0 + u * (256 / P)][i];
                }
            } else {
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    const int row = t * TR + lr0 + u * (256 / P);
                    const size_t e = static_cast<size_t>(row) * P + i;
                    const bool ok = row < n;
                    dv[u] = ok ? D[e] : 0.0;
                    qv[u] = ok ? Q[e] : 0.0;
                    xv[u] = ok ? X[e] : 0.0;
                    rv[u] = ok ? R[e] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < RP; ++u) {
                    td_[lr0 + u * (256 / P)][i] = dv[u];
                    tq_[lr0 + u * (256 / P)][i] = qv[u];
                }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int lr = lr0 + u * (256 / P);
                const int row = t * TR + lr;
                const size_t e = static_cast<size_t>(row) * P + i;
                double rnew = 0.0;
                if (row < n && i < p) {
                    double x = xv[u];
                    for (int jj = 0; jj < p; ++jj) x = fma(al[i][jj], td_[lr][jj], x);
                    X[e] = x;
                    double r = rv[u];
                    for (int jj = 0; jj < p; ++jj) r = fma(al[i][jj], tq_[lr][jj], r);
                    R[e] = r;
                    rnew = r;
                    nrm = fma(r, r, nrm);
                }
                tr_[lr][i] = rnew;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const int lr = lr0 + u * (256 / P);
                const int row = t * TR + lr;
                double dn = 0.0;
                if (row < n && i < p) {
                    dn = tr_[lr][i];
                    for (int jj = 0; jj < p; ++jj) dn = fma(be[i][jj], td_[lr][jj], dn);
                }
                if (row < n) Dn[static_cast<size_t>(row) * P + i] = dn;
                tdn[lr][i] = dn;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (pi[q] >= 0) {
                    double sp = part[q];
                    for (int r = pg[q]; r < TR; r += GR) sp = fma(tdn[r][pi[q]], tdn[r][pj[q]], sp);
                    part[q] = sp;
                }
            __syncthreads();
        }
        nred[tid] = nrm;
        __syncthreads();
        if (tid < P) {
            double sn = 0.0;
            for (int r = 0; r < 256 / P; ++r) sn += nred[r * P + tid];
            norm_part[static_cast<size_t>(blockIdx.x) * P + tid] = sn;
        }
#ifdef COOPCG_PHASE_TIMES
        PHASE_MARK(7);
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_phase_ns[7], 1ull);
#endif
        if (GR == 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
                if (pi[q] >= 0) pair_part[static_cast<size_t>(blockIdx.x) * npairs + tid + q * 256] = part[q];
        } else {
            __syncthreads();
            nred[tid] = part[0];
            __syncthreads();
            if (tid < npairs) {
                double sp = 0.0;
                for (int g = 0; g < GR; ++g) sp += nred[tid * GR + g];
                pair_part[static_cast<size_t>(blockIdx.x) * npairs + tid] = sp;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// (5) Norms from partials -> record + convergence (the fast twin of the tail of
// beta_solve_warp; solvers.hpp:125-154).  `diag_stride` selects the layout:
// norm partials are P values per CTA (stride P), residual-pass partials keep
// the squared norms on the diagonal of G1 (offset P*P, stride P+1).
__global__ void __launch_bounds__(256)
    fast_record_kernel(const double* __restrict__ part, int nparts, int part_stride, int part_off, int diag_stride,
                       double* __restrict__ small, Ctl* ctl, double* __restrict__ tr_norms,
                       double* __restrict__ tr_minres, unsigned long long* __restrict__ tr_wall, int capacity) {
    pdl_wait();
    if (*reinterpret_cast<volatile int*>(&ctl->stop)) return;
    __shared__ double norms[kMaxP], sums[kMaxP], red[256];
    const int p = ctl->p, P = ctl->P;
    const SmallLayout L{P};
    const int tid = threadIdx.x;
    cta_reduce_fixed(part, nparts, part_stride, part_off, diag_stride, p, sums, red);
    if (tid < p) {
        const double s = sums[tid];
        small[L.nsq_r() + tid] = s;
        norms[tid] = sqrt(s);
        small[L.norm() + tid] = norms[tid];
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned long long now = globaltimer_ns();
        const int k = ctl->k;
        double m = norms[0];
        int slot = -1;
        for (int j = 0; j < p; ++j) {
            m = (norms[j] < m) ? norms[j] : m;
            if (slot < 0 && norms[j] <= ctl->tol) slot = j;
        }
        if (k < capacity) {
            const int p0 = ctl->p0;
            for (int j = 0; j < p0; ++j) tr_norms[static_cast<size_t>(k) * p0 + j] = __longlong_as_double(0x7ff8000000000000ll);
            for (int j = 0; j < p; ++j) tr_norms[static_cast<size_t>(k) * p0 + ctl->ids[j]] = norms[j];
            tr_minres[k] = m;
            tr_wall[k] = now - ctl->t_last;
        }
        ctl->t_last = now;
        ctl->iterations = k + 1;
        if (slot >= 0) {
            ctl->status = 0;
            ctl->converged_agent = ctl->ids[slot];
            ctl->stop = 1;
        }
    }
}

// Initial / final norms from residual-pass partials (diag of G1).
__global__ void fast_norms_kernel(const double* __restrict__ part, int nparts, int part_stride, int part_off,
                                  int diag_stride, Ctl* ctl, double* __restrict__ out, int setup,
                                  double* __restrict__ small) {
    __shared__ double nv[kMaxP], sums[kMaxP], red[256];
    const int p = ctl->p;
    const SmallLayout L{ctl->P};
    const int tid = threadIdx.x;
    cta_reduce_fixed(part, nparts, part_stride, part_off, diag_stride, p, sums, red);
    if (tid < p) {
        const double s = sums[tid];
        nv[tid] = sqrt(s);
        out[tid] = nv[tid];
        if (setup) {
            small[L.nsq_r() + tid] = s;
            small[L.norm() + tid] = nv[tid];
        }
    }
    __syncthreads();
    if (tid == 0) {
        double m = nv[0];
        int slot = -1;
        for (int j = 0; j < p; ++j) {
            m = (nv[j] < m) ? nv[j] : m;
            if (slot < 0 && nv[j] <= ctl->tol) slot = j;
        }
        out[p] = m;
        if (setup) {
            if (slot >= 0 && ctl->algo == 0) {
                ctl->status = 0;
                ctl->converged_agent = slot;
                ctl->stop = 1;
            }
            ctl->t_last = globaltimer_ns();
        }
    }
}

} // namespace coopcg_gpu
