// gen_kernels.cuh -- on-device generators for the BASELINE inputs.
//
// The reference has no generator for the BASELINE configs; these follow the
// spec in DESIGN.md §3 built on the reference's counter-based SplitMix64
// streams (coopcg/rng.hpp:16-20, :35-48, :80-87).  Every value is a pure
// function of (seed, element index) or a sequential chain with the
// specified order, so the GPU bytes equal the host oracle's bytes
// (tests/test_gpu_parity.py).  A is written in the panel layout of
// common.cuh (ap_idx) for the context's rows.
#pragma once
#include "common.cuh"

namespace coopcg_gpu {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t id, uint64_t extra) {
    return mix64(seed ^ mix64(id ^ mix64(extra)));
}
__device__ __forceinline__ double uniform_pm1_dev(uint64_t key, uint64_t c) {
    const uint64_t x = mix64(key + c * kGolden);
    const double u = __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
    return __dadd_rn(-1.0, __dmul_rn(2.0, u));
}

// Off-diagonal entries of the diagonally dominant matrix: A_ij = A_ji =
// (B_lo,hi + B_hi,lo) / 2 with B_ij ~ U[-1,1] at counter i*n + j + 1.
// Iterates over storage order (coalesced writes for either layout).
__global__ void gen_dd_offdiag_kernel(double* __restrict__ Ap, ALay L, int n, int n_loc, int row0, uint64_t key,
                                      size_t total) {
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        int k, il;
        a_decode(L, n, e, k, il);
        double v = 0.0;
        const uint64_t i = static_cast<uint64_t>(row0 + il), kk = static_cast<uint64_t>(k);
        if (il < n_loc && k < n && kk != i) {
            const uint64_t lo = kk < i ? kk : i, hi = kk < i ? i : kk;
            const uint64_t un = static_cast<uint64_t>(n);
            const double u1 = uniform_pm1_dev(key, lo * un + hi + 1);
            const double u2 = uniform_pm1_dev(key, hi * un + lo + 1);
            v = __dmul_rn(__dadd_rn(u1, u2), 0.5);
        }
        Ap[e] = v;
    }
}

// Diagonal: A_ii = (sum_{j != i, ascending} |A_ij|) + 1.  One chain per row.
__global__ void gen_dd_diag_kernel(double* __restrict__ Ap, ALay L, int n, int n_loc, int row0) {
    const int il = blockIdx.x * blockDim.x + threadIdx.x;
    if (il >= n_loc) return;
    const int i = row0 + il;
    double acc = 0.0;
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
        const double a = fabs(Ap[a_idx(L, n, j, il)]);
        if (j != i) acc = __dadd_rn(acc, a);
    }
    Ap[a_idx(L, n, i, il)] = __dadd_rn(acc, 1.0);
}

// Householder construction on the context's rows [row0, row0 + n_loc):
// M = diag(lambda); for r = m-1 .. 0: M <- H_r M H_r with
//   s = v.v, w = M v, c = v.w, t1 = 2/s, t2 = (4 c)/(s s),
//   M_ij <- (M_ij - t1 (v_i w_j + w_i v_j)) + t2 (v_i v_j)
// (every sum sequential ascending, one rounding per op).  Row i of w needs
// only row i of M, the update of row i needs all of w: a row-sharded context
// computes its rows of w, the caller all-gathers w, every rank forms s, c
// from the full vectors identically and updates its own rows.
__global__ void hh_init_kernel(double* __restrict__ Ap, ALay L, int n, int n_loc, int row0,
                               const double* __restrict__ lambda, size_t total) {
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        int k, il;
        a_decode(L, n, e, k, il);
        const int i = row0 + il;
        Ap[e] = (il < n_loc && k < n && i == k) ? lambda[i] : 0.0;
    }
}
// w[row0 + il] = sum_k M(il, k) v[k], k ascending
__global__ void hh_w_kernel(const double* __restrict__ Ap, ALay L, int n, int n_loc, int row0,
                            const double* __restrict__ v, double* __restrict__ w) {
    const int il = blockIdx.x * blockDim.x + threadIdx.x;
    if (il >= n_loc) return;
    double acc = 0.0;
#pragma unroll 4
    for (int k = 0; k < n; ++k) acc = mac_exact(acc, Ap[a_idx(L, n, k, il)], v[k]);
    w[row0 + il] = acc;
}
__global__ void hh_scalars_kernel(int n, const double* __restrict__ v, const double* __restrict__ w,
                                  double* __restrict__ t12) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0, c = 0.0;
    for (int k = 0; k < n; ++k) s = mac_exact(s, v[k], v[k]);
    for (int k = 0; k < n; ++k) c = mac_exact(c, v[k], w[k]);
    t12[0] = __ddiv_rn(2.0, s);
    t12[1] = __ddiv_rn(__dmul_rn(4.0, c), __dmul_rn(s, s));
}
__global__ void hh_update_kernel(double* __restrict__ Ap, ALay L, int n, int n_loc, int row0,
                                 const double* __restrict__ v, const double* __restrict__ w,
                                 const double* __restrict__ t12, size_t total) {
    const double t1 = t12[0], t2 = t12[1];
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        int k, il;
        a_decode(L, n, e, k, il);
        if (il >= n_loc || k >= n) continue;
        const int i = row0 + il;
        // element (i, k); the expression is symmetric in (i, k) bit for bit.
        const double q = __dadd_rn(__dmul_rn(v[i], w[k]), __dmul_rn(w[i], v[k]));
        const double m1 = __dsub_rn(Ap[e], __dmul_rn(t1, q));
        Ap[e] = __dadd_rn(m1, __dmul_rn(t2, __dmul_rn(v[i], v[k])));
    }
}

} // namespace coopcg_gpu
