// verify_kernels.cuh -- the reference's verification mode on the device:
// SolveOptions::x_star (A-norm error per agent and iteration,
// coopcg/block_cg.hpp:316-331 + coopcg/dense_ops.hpp:159-196) and
// SolveOptions::keep_history (X_k, R_k, D_k blocks, coopcg/solvers.hpp:43-50).
// Off the hot path: one extra A.D per iteration when x_star is set.
#pragma once
#include "common.cuh"

namespace coopcg_gpu {

// E[:, j] = X[:, j] - x*  (block_cg.hpp:322-327); padded columns stay zero.
__global__ void ver_diff_kernel(const double* __restrict__ X, const double* __restrict__ xs,
                                double* __restrict__ E, int n, int p, int P) {
    const size_t total = static_cast<size_t>(n) * P;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t i = e / P;
        const int j = static_cast<int>(e % P);
        E[e] = (j < p) ? __dsub_rn(X[e], xs[i]) : 0.0;
    }
}

// Dn = R + D beta^T, j ascending from the base value (block_cg.hpp:270-273,
// kernels.hpp:36-49), beta row-major with row stride P; sd: Dn = R.
__global__ void ver_direction_kernel(const double* __restrict__ R, const double* __restrict__ D,
                                     const double* __restrict__ beta, double* __restrict__ Dn, int n, int p, int P,
                                     int sd) {
    const size_t total = static_cast<size_t>(n) * P;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t row = e / P;
        const int i = static_cast<int>(e % P);
        double v = 0.0;
        if (i < p) {
            v = R[e];
            if (!sd)
                for (int j = 0; j < p; ++j) v = __dadd_rn(v, __dmul_rn(beta[i * P + j], D[row * P + j]));
        }
        Dn[e] = v;
    }
}

// out[j] = a_norm(A, e_j) from e_j and A e_j: q = dot(e_j, A e_j) summed
// sequentially from +0.0 with separately rounded products (kernels.hpp:20-26),
// sqrt(q) for q >= 0; a negative q within 1e-12 * sum |e_i| |(A e)_i| is
// clamped to 0, beyond it raises *flag (dense_ops.hpp:175-196:
// SpdViolationError).  One CTA; thread j < p owns agent j's chain, all threads
// stage the row tiles through shared memory.
constexpr int kVerTile = 64;
__global__ void __launch_bounds__(256)
    ver_anorm_kernel(const double* __restrict__ E, const double* __restrict__ AE, int n, int p, int P,
                     double* __restrict__ out, int* __restrict__ flag) {
    extern __shared__ double ver_sm[];
    double* se = ver_sm;
    double* sa = ver_sm + kVerTile * P;
    const int j = threadIdx.x;
    double acc = 0.0;
    for (int i0 = 0; i0 < n; i0 += kVerTile) {
        const int rows = min(kVerTile, n - i0);
        for (int t = threadIdx.x; t < rows * P; t += blockDim.x) {
            se[t] = E[static_cast<size_t>(i0) * P + t];
            sa[t] = AE[static_cast<size_t>(i0) * P + t];
        }
        __syncthreads();
        if (j < p)
            for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, __dmul_rn(se[r * P + j], sa[r * P + j]));
        __syncthreads();
    }
    if (j < p) {
        double res = 0.0;
        if (acc < 0.0) {
            double scale = 0.0;
            for (int i = 0; i < n; ++i)
                scale = __dadd_rn(scale, __dmul_rn(fabs(E[static_cast<size_t>(i) * P + j]),
                                                   fabs(AE[static_cast<size_t>(i) * P + j])));
            if (acc < __dmul_rn(-1e-12, scale)) atomicExch(flag, 1);
        } else {
            res = __dsqrt_rn(acc);
        }
        out[j] = res;
    }
}

}  // namespace coopcg_gpu
