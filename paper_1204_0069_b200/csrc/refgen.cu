// refgen.cu -- the reference's own problem family generated on the device,
// bit-identical to the reference.
//
//   make_problem<double>(ProblemSpec{n, p, cond, seed})   problem.hpp:219-230
//     A  = random_spd_with_spectrum(n, cond, seed).A       problem.hpp:118-152
//          U = haar_orthogonal(n, seed)                    problem.hpp:65-108
//          A = (U Lambda) U^T, then SpdMatrix symmetrises  dense.hpp:112-122
//     b, X0 = random_rhs_and_starts(n, p, seed)            problem.hpp:187-200
//
// haar_orthogonal is modified Gram-Schmidt in a fixed order: for column j,
// for i < j: coef = sum_r u_i[r] v[r] (sequential r), v -= coef u_i; then
// nsq = sum_r v[r]^2, v /= sqrt(nsq).  The GPU keeps that order per column and
// runs every column's chain concurrently, one wavefront step per basis vector:
//   N(t): column t takes its pending projection onto u_{t-1}, sums its square
//         norm (one sequential chain), and is normalised -> u_t   (1 CTA)
//   P(t): every column j > t takes its pending projection onto u_{t-1} and
//         sums coef_{j,t} = u_t . v_j (one chain per column)       (1 warp / 32 cols)
// so column j sees exactly the reference's operation sequence.  W (the
// Gaussian sample, overwritten by U) is stored in 32-column blocks (wcb), so
// a P warp's 32 columns x 128 rows are one 32 KB bulk copy through a 6-stage
// ring.  U Lambda U^T is an n^3 product with a sequential k-chain per entry
// (acc += (u_ik * l_k) * u_jk, k ascending).
// The Gaussians come from glibc log/cos on the host (CUDA's are not
// bit-identical to glibc) and are uploaded once, like the Householder vectors
// of the BASELINE generator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/coopcg_gpu.h"
#include "common.cuh"
#include "host_rng.h"

namespace coopcg_gpu {

constexpr int kMgsTR = 32;   // rows per pipelined sub-tile
constexpr int kMgsSR = 128;  // rows per ring stage (one bulk copy)
constexpr int kMgsS = 6;     // ring stages (one CTA per SM)
constexpr int kMgsS2 = 3;    // ring stages when the grid exceeds the SMs (two CTAs per SM)
constexpr int kMgsStage = kMgsSR * 32 + 2 * kMgsSR;  // doubles: W rows + u_{t-1} + u_t
constexpr size_t mgs_smem(int stages) { return sizeof(double) * stages * kMgsStage; }
constexpr int kNormSmemMaxN = 24576;  // above this N(t) keeps the squares in global scratch

// Column-block layout of the Gram-Schmidt working matrix W (n x n, np = n
// rounded up to 32): block jb holds columns 32 jb .. 32 jb + 31 for all np
// rows, row-major inside the block, so a P stage (128 rows x 32 columns) is
// one contiguous 32 KB run (one bulk copy) and column t is a 256-byte stride.
// (A 9.5 KB gap between blocks, tried against HBM channel camping of the
// ~100 concurrent block streams, changed nothing: kWcbPad = 0.)
constexpr int kWcbPad = 0;
__host__ __device__ __forceinline__ size_t wcb_stride(int np) { return static_cast<size_t>(np) * 32 + kWcbPad; }
__host__ __device__ __forceinline__ size_t wcb(int np, int r, int j) {
    return static_cast<size_t>(j >> 5) * wcb_stride(np) + (static_cast<size_t>(r) << 5) + static_cast<size_t>(j & 31);
}

// N(t): v = W[:, t] (- coef[t] * u_{t-1}), nsq = sum_r v_r * v_r (r ascending,
// problem.hpp:87-89), norm = sqrt(nsq), u_t = v / norm (problem.hpp:98-99).
// W is in the column-block layout (wcb); u vectors are zero-padded to np rows.
// All threads form v (kept in uout) and the squares (shared memory, or the
// global scratch pg for n > kNormSmemMaxN); thread 0 then runs the one
// sequential chain over the squares in 16-step batches.
__global__ void __launch_bounds__(512) mgs_norm_kernel(double* __restrict__ W, int n, int np, int t,
                                                        const double* __restrict__ coef,
                                                        const double* __restrict__ uprev, double* __restrict__ uout,
                                                        double* __restrict__ pg, int* __restrict__ err) {
    extern __shared__ __align__(16) double sq[];
    __shared__ double s_norm;
    pdl_wait();
    pdl_trigger();
    const double* col = W + wcb(np, 0, t);  // element r at col[32 r]
    double* pr = pg ? pg : sq;
    const double c = t > 0 ? coef[t] : 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double x = col[32 * r];
        if (t > 0) x = __dsub_rn(x, __dmul_rn(c, uprev[r]));  // v[r] -= coef * u[r]
        uout[r] = x;
        pr[r] = __dmul_rn(x, x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        int r = 0;
        if (!pg) {  // shared memory, 16 squares per batch (8.8 cycles/step, profiles/r01_probe_chain_split.txt)
            const double2* p2 = reinterpret_cast<const double2*>(sq);
            const int nb = n / 16;
            for (int b = 0; b < nb; ++b) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = p2[b * 8 + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __dadd_rn(acc, v[u].x);
                    acc = __dadd_rn(acc, v[u].y);
                }
            }
            r = nb * 16;
        }
        for (; r < n; ++r) acc = __dadd_rn(acc, pr[r]);
        s_norm = __dsqrt_rn(acc);
    }
    __syncthreads();
    const double nrm = s_norm;
    if (nrm == 0.0) {  // measure-zero degenerate draw (the reference re-draws, problem.hpp:91-97)
        if (threadIdx.x == 0) atomicCAS(err, 0, t + 1);
        return;
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double u = __ddiv_rn(uout[r], nrm);
        uout[r] = u;
        W[wcb(np, r, t)] = u;
    }
}

// P(t): columns j in (t, n) in blocks of 32 (one one-warp CTA per block,
// lane = column): apply the pending projection v_j -= coef_{j,t-1} u_{t-1}
// (problem.hpp:85-86) and sum coef_{j,t} = sum_r u_t[r] * v_j[r]
// (problem.hpp:81-84), r ascending.  Stages of 128 rows x 32 columns (+ the
// two u slices) arrive as one 32 KB bulk copy each through a 6-stage ring on
// mbarriers (few large copies: 8 KB copies streamed at ~7 GB/s per CTA);
// updated values go straight back from registers (one coalesced 256-byte row
// store per step).  Software-pipelined by 32-row sub-tiles: step rr adds
// sub-tile g's product rr to the chain and forms sub-tile g+1's row rr
// (update, store, product), so the dependent DADD chain overlaps the
// independent work.  Lanes outside (t, n) (first / last block) use c = 0 and
// never store; their sums are discarded.
template <bool PEND, int S>
__global__ void __launch_bounds__(32) mgs_proj_kernel(double* __restrict__ W, int n, int np, int t,
                                                      double* __restrict__ coef, const double* __restrict__ uprev,
                                                      const double* __restrict__ ucur) {
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t full[S];
    constexpr int TR = kMgsTR, SR = kMgsSR, SUB = SR / TR, STAGE = kMgsStage, AHEAD = S - 1;
    const int lane = threadIdx.x;
    const int jb = ((t + 1) >> 5) + blockIdx.x;
    const int j = jb * 32 + lane;
    const bool valid = j > t && j < n;
    double* gblk = W + wcb(np, 0, jb * 32);
    const int ntiles = (n + TR - 1) / TR;
    const int nstages = (n + SR - 1) / SR;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const double c = (PEND && valid) ? coef[j] : 0.0;
    const bool store = PEND && valid;

    // stage q: rows q*SR .. q*SR + SR - 1 (the allocation is padded past n)
    auto issue = [&](int q) {
        if (q >= nstages || lane != 0) return;
        const int s = q % S;
        double* st = ring + s * STAGE;
        const int r0 = q * SR;
        mbar_arrive_expect_tx(&full[s], SR * 256 + 2 * SR * 8);
        bulk_g2s(st, gblk + static_cast<size_t>(r0) * 32, SR * 256, &full[s]);
        bulk_g2s(st + SR * 32, uprev + r0, SR * 8, &full[s]);
        bulk_g2s(st + SR * 32 + SR, ucur + r0, SR * 8, &full[s]);
    };
    // row rr of sub-tile g: x = v (- c u_{t-1}), stored back; returns u_t * x
    auto row = [&](int g, int rr) {
        const double* st = ring + (g / SUB % S) * STAGE;
        const int o = (g % SUB) * TR + rr;
        double x = st[o * 32 + lane];
        if (PEND) {
            x = __dsub_rn(x, __dmul_rn(c, st[SR * 32 + o]));
            // st.global (not a generic store): a generic store may alias the
            // shared ring, which would hold every later ring load behind it
            if (store) __stcg(gblk + (static_cast<size_t>(g) * TR + rr) * 32 + lane, x);
        }
        return __dmul_rn(st[SR * 32 + SR + o], x);
    };

    for (int q = 0; q < S; ++q) issue(q);  // stage q + AHEAD refills slot (q - 1) % S from stage 1 on
    double pr[TR];
    mbar_wait(&full[0], 0);
#pragma unroll
    for (int rr = 0; rr < TR; ++rr) pr[rr] = row(0, rr);
    __syncwarp();
    double acc = 0.0;
    for (int g = 0; g + 1 < ntiles; ++g) {  // every sub-tile but the last is full
        const int ng = g + 1;
        if (ng % SUB == 0) {
            const int q = ng / SUB;
            issue(q + AHEAD);  // refills the stage whose last sub-tile was formed last iteration
            mbar_wait(&full[q % S], (q / S) & 1);
        }
#pragma unroll
        for (int rr = 0; rr < TR; ++rr) {
            acc = __dadd_rn(acc, pr[rr]);
            pr[rr] = row(ng, rr);
        }
        __syncwarp();
    }
    const int rows = n - (ntiles - 1) * TR;
#pragma unroll
    for (int rr = 0; rr < TR; ++rr)
        if (rr < rows) acc = __dadd_rn(acc, pr[rr]);
    if (valid) coef[j] = acc;
}

// a_ij = sum_k (u_ik * lambda_k) * u_jk, k ascending from +0.0
// (problem.hpp:141-147), written to A(i, j) of the context layout.
constexpr int kGB = 64, kGK = 16;
__global__ void __launch_bounds__(256) spd_product_kernel(const double* __restrict__ U, const double* __restrict__ lam,
                                                          int n, int np, double* __restrict__ At, ALay L) {
    __shared__ double Ws[kGK][kGB + 1];
    __shared__ double Us[kGK][kGB + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int i0 = blockIdx.y * kGB, j0 = blockIdx.x * kGB;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < n; k0 += kGK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + 256 * q, ii = e >> 4, kk = e & 15, k = k0 + kk;
            const int gi = i0 + ii, gj = j0 + ii;
            Ws[kk][ii] = (gi < n && k < n) ? __dmul_rn(U[wcb(np, gi, k)], lam[k]) : 0.0;
            Us[kk][ii] = (gj < n && k < n) ? U[wcb(np, gj, k)] : 0.0;
        }
        __syncthreads();
        const int kmax = min(kGK, n - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            double wa[4], ub[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) wa[a] = Ws[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) ub[b] = Us[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(wa[a], ub[b]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int i = i0 + ty + 16 * a, jj = j0 + tx + 16 * b;
            if (i < n && jj < n) At[a_idx(L, n, jj, i)] = acc[a][b];
        }
}

// SpdMatrix float-mode symmetrisation (dense.hpp:115-122): for i < j,
// A(i,j) = A(j,i) = (A(i,j) + A(j,i)) / 2.0; the diagonal is untouched.
__global__ void spd_symmetrize_kernel(double* __restrict__ At, ALay L, int n) {
    const size_t total = static_cast<size_t>(n) * n;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
        if (i >= j) continue;
        const size_t ij = a_idx(L, n, j, i), ji = a_idx(L, n, i, j);
        const double avg = __ddiv_rn(__dadd_rn(At[ij], At[ji]), 2.0);
        At[ij] = avg;
        At[ji] = avg;
    }
}

// ---- host side ---------------------------------------------------------------

// random_spd_with_spectrum's spectrum (problem.hpp:125-139): lambda_i ~
// uniform(1, cond) from the `spectrum` stream, first minimum -> 1, first
// maximum -> cond (front/back when all draws are equal).
void random_spd_spectrum(int n, double cond, uint64_t seed, double* lambda) {
    for (int i = 0; i < n; ++i) lambda[i] = 1.0;
    if (n < 2) return;
    const uint64_t key = host_rng::key(seed, 2, 0);
    for (int i = 0; i < n; ++i) lambda[i] = host_rng::uniform(key, (uint64_t)i + 1, 1.0, cond);
    double* lo = std::min_element(lambda, lambda + n);
    double* hi = std::max_element(lambda, lambda + n);
    if (lo == hi) {
        lambda[0] = 1.0;
        lambda[n - 1] = cond;
    } else {
        *lo = 1.0;
        *hi = cond;
    }
}

// Gaussian sample of haar_orthogonal (problem.hpp:74-79): column j, row i is
// normal number j*n + i of the `orthogonal` stream; stored row-major.
static void haar_gaussians(int n, int np, uint64_t seed, double* Wcb) {
    const uint64_t key = host_rng::key(seed, 1, 0);
    unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 64u));
    if ((size_t)n * n < (1u << 16)) nt = 1;
    auto work = [&](unsigned w) {
        for (int i = (int)w; i < n; i += (int)nt)
            for (int j = 0; j < n; ++j)
                Wcb[wcb(np, i, j)] = host_rng::normal(key, (uint64_t)j * (uint64_t)n + (uint64_t)i);
    };
    if (nt == 1) {
        work(0);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nt; ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
}

// Device part.  At: the context's A storage (layout L, ap_elems doubles, the
// full n x n matrix).  Returns a coopcg_err; msg explains failures.
int refgen_random_spd(double* At, ALay L, size_t ap_elems, int n, double cond, uint64_t seed, cudaStream_t st,
                      std::string& msg) {
    if (n < 2) {
        msg = "random_spd: the device generator needs n >= 2";
        return COOPCG_E_DIMENSION;
    }
    if (!(cond >= 1.0)) {
        msg = "random_spd: condition number must be >= 1";  // problem.hpp:122-123
        return COOPCG_E_INVALID;
    }
    std::vector<double> lam(n);
    random_spd_spectrum(n, cond, seed, lam.data());
    // W in the column-block layout, np = n rounded up to 32 (rows and
    // columns); the padding is zero and never enters a chain.
    const int np = (n + 31) & ~31;
    const size_t wel = (size_t)(np / 32) * wcb_stride(np) + (size_t)kMgsSR * 32;  // + the last stage's over-read
    std::vector<double> Wh(wel, 0.0);
    haar_gaussians(n, np, seed, Wh.data());

    double *W = nullptr, *dl = nullptr, *coef = nullptr, *ubuf = nullptr, *vg = nullptr;
    int* derr = nullptr;
    cudaError_t e = cudaSuccess;
    auto cleanup = [&]() {
        cudaFree(W);
        cudaFree(dl);
        cudaFree(coef);
        cudaFree(ubuf);
        cudaFree(vg);
        cudaFree(derr);
    };
#define RG(call)                                                                                   \
    do {                                                                                           \
        e = (call);                                                                                \
        if (e != cudaSuccess) {                                                                    \
            msg = std::string("random_spd: ") + #call + ": " + cudaGetErrorString(e);              \
            cleanup();                                                                             \
            return COOPCG_E_CUDA;                                                                  \
        }                                                                                          \
    } while (0)
    RG(cudaMalloc(&W, sizeof(double) * wel));
    RG(cudaMalloc(&dl, sizeof(double) * n));
    RG(cudaMalloc(&coef, sizeof(double) * np));
    RG(cudaMalloc(&ubuf, sizeof(double) * (2 * np + kMgsSR)));
    RG(cudaMalloc(&derr, sizeof(int)));
    // (tests force the global-scratch path at small n)
    const bool norm_in_smem = n <= kNormSmemMaxN && std::getenv("COOPCG_REFGEN_NORM_GLOBAL") == nullptr;
    if (!norm_in_smem) RG(cudaMalloc(&vg, sizeof(double) * n));
    RG(cudaMemcpyAsync(W, Wh.data(), sizeof(double) * wel, cudaMemcpyHostToDevice, st));
    RG(cudaMemcpyAsync(dl, lam.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    RG(cudaMemsetAsync(coef, 0, sizeof(double) * np, st));
    RG(cudaMemsetAsync(ubuf, 0, sizeof(double) * (2 * np + kMgsSR), st));
    RG(cudaMemsetAsync(derr, 0, sizeof(int), st));
    const size_t norm_smem = norm_in_smem ? sizeof(double) * n : 0;
    RG(cudaFuncSetAttribute(mgs_norm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)norm_smem));
    RG(cudaFuncSetAttribute(mgs_proj_kernel<false, kMgsS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mgs_smem(kMgsS)));
    RG(cudaFuncSetAttribute(mgs_proj_kernel<true, kMgsS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mgs_smem(kMgsS)));
    RG(cudaFuncSetAttribute(mgs_proj_kernel<false, kMgsS2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mgs_smem(kMgsS2)));
    RG(cudaFuncSetAttribute(mgs_proj_kernel<true, kMgsS2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mgs_smem(kMgsS2)));
    const bool force_two = std::getenv("COOPCG_REFGEN_TWO_PER_SM") != nullptr;  // tests: the 3-stage variant at small n
    int nsm = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }

    // Programmatic dependent launch: each step's kernel is scheduled while the
    // previous one drains and waits (griddepcontrol.wait) for its results.
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg_n{}, cfg_p{};
    cfg_n.gridDim = dim3(1);
    cfg_n.blockDim = dim3(512);
    cfg_n.dynamicSmemBytes = norm_smem;
    cfg_n.stream = st;
    cfg_n.attrs = attr;
    cfg_n.numAttrs = 1;
    cfg_p = cfg_n;
    cfg_p.blockDim = dim3(32);
    for (int t = 0; t < n; ++t) {
        double* uprev = ubuf + (size_t)((t + 1) & 1) * np;  // u_{t-1}
        double* ucur = ubuf + (size_t)(t & 1) * np;          // u_t
        RG(cudaLaunchKernelEx(&cfg_n, mgs_norm_kernel, W, n, np, t, (const double*)coef, (const double*)uprev, ucur,
                              vg, derr));
        if (t + 1 < n) {
            const int blocks = (n + 31) / 32 - (t + 1) / 32;
            cfg_p.gridDim = dim3((unsigned)blocks);
            // more column blocks than SMs: a 3-stage ring so two CTAs share an SM (one wave)
            const bool two = blocks > nsm || force_two;
            cfg_p.dynamicSmemBytes = mgs_smem(two ? kMgsS2 : kMgsS);
            auto kern = t == 0 ? (two ? mgs_proj_kernel<false, kMgsS2> : mgs_proj_kernel<false, kMgsS>)
                               : (two ? mgs_proj_kernel<true, kMgsS2> : mgs_proj_kernel<true, kMgsS>);
            RG(cudaLaunchKernelEx(&cfg_p, kern, W, n, np, t, coef, (const double*)uprev, (const double*)ucur));
        }
    }
    RG(cudaMemsetAsync(At, 0, sizeof(double) * ap_elems, st));
    dim3 grid((n + kGB - 1) / kGB, (n + kGB - 1) / kGB);
    spd_product_kernel<<<grid, 256, 0, st>>>(W, dl, n, np, At, L);
    RG(cudaGetLastError());
    spd_symmetrize_kernel<<<148 * 8, 256, 0, st>>>(At, L, n);
    RG(cudaGetLastError());
    int herr = 0;
    RG(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st));
    RG(cudaStreamSynchronize(st));
#undef RG
    cleanup();
    if (herr) {
        msg = "random_spd: zero-norm Gaussian column " + std::to_string(herr - 1) +
              " (measure-zero draw the reference re-samples; not supported on the device)";
        return COOPCG_E_NUMERICAL_BREAKDOWN;
    }
    return COOPCG_OK;
}

}  // namespace coopcg_gpu

extern "C" {

int coopcg_gen_random_spd_spectrum(int n, double cond, uint64_t seed, double* lambda) {
    if (n < 1 || !lambda || !(cond >= 1.0)) return COOPCG_E_INVALID;
    coopcg_gpu::random_spd_spectrum(n, cond, seed, lambda);
    return COOPCG_OK;
}

// random_rhs_and_starts<double> (problem.hpp:187-200): b_i = uniform(-10, 10)
// draw i+1 of the `rhs` stream; X0(i, j) = draw j*n + i + 1 of `starts`.
int coopcg_gen_reference_rhs_starts(int n, int p, uint64_t seed, double* b, double* X0) {
    using namespace coopcg_gpu;
    if (n < 1 || p < 1 || !b || !X0) return COOPCG_E_INVALID;
    const uint64_t kr = host_rng::key(seed, 3, 0), ks = host_rng::key(seed, 4, 0);
    for (int i = 0; i < n; ++i) b[i] = host_rng::uniform(kr, (uint64_t)i + 1, -10.0, 10.0);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i)
            X0[(size_t)j * n + i] = host_rng::uniform(ks, (uint64_t)j * (uint64_t)n + (uint64_t)i + 1, -10.0, 10.0);
    return COOPCG_OK;
}

}  // extern "C"
