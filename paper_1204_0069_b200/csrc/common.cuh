// common.cuh -- shared device definitions for the cCG hot path (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace coopcg_gpu {

constexpr int kMaxP = 32;

// Offsets into the per-context "small" array (p x p grids stored with row
// stride P, per-agent vectors of length P).  Row-major like the reference's
// gram/rhs/alpha/beta grids (block_cg.hpp:45-46).
struct SmallLayout {
    int P;
    __host__ __device__ int raw() const { return 0; }
    __host__ __device__ int rhs_a() const { return P * P; }
    __host__ __device__ int rhs_b() const { return 2 * P * P; }
    __host__ __device__ int alpha() const { return 3 * P * P; }
    __host__ __device__ int beta() const { return 4 * P * P; }
    __host__ __device__ int nsq_d() const { return 5 * P * P; }
    __host__ __device__ int nsq_r() const { return 5 * P * P + P; }
    __host__ __device__ int nsq_f() const { return 5 * P * P + 2 * P; }
    __host__ __device__ int norm() const { return 5 * P * P + 3 * P; }
    __host__ __device__ int mgs() const { return 5 * P * P + 4 * P; } // P values
    __host__ __device__ int total() const { return 5 * P * P + 5 * P; }
};

// Peer-memory row push (row-sharded contexts, one process per GPU): the
// kernel that produces this rank's rows of Q also stores them into every
// rank's copy of Q (CUDA IPC mappings over NVLink; dst[self] is the local
// buffer), so no separate all-gather of Q is needed.  n == 0: local only.
constexpr int kMaxPeers = 8;
struct PeerRows {
    double* dst[kMaxPeers];
    int n;
};

// Device control block: the coordinator state of DriverControl
// (block_cg.hpp:106-125) plus the factorisation shared by the alpha and beta
// solves (the reference re-factors the same Gram matrix per agent, with
// identical results; SURVEY §8a notes).
struct Ctl {
    int stop;             // every kernel becomes a no-op once set
    int status;           // coopcg_status
    int err;              // coopcg_err raised inside the loop (SPD violation)
    int err_iter;
    int k;                // current iteration index
    int iterations;       // IterationRecords written
    int converged_agent;
    int need_exact_rank;  // rank certificate inconclusive -> exact MGS this iteration
    int force_exact;      // tests: always run the exact MGS
    int exact_rank_checks;
    int rank_result;
    int perm[kMaxP];
    double lu[kMaxP * kMaxP];
    unsigned long long t_last;
    // options (SolveOptions)
    double tol;
    double rank_rel_tol;
    int max_iters;
    int p;                // active agents
    int P;
    int algo;             // 0 ccg, 1 mccg (restriction allowed)
    int p0;               // agents at the start (trace row width)
    int restrict_pending; // mccg: rank drop seen; device paused for the host to restrict
    int rank_cols[kMaxP]; // pivot columns of the last exact MGS (dense_ops.hpp:254-256)
    int ids[kMaxP];       // original agent id of each active slot (block_cg.hpp:48)
};

// One sequential dot-product chain (kernels.hpp:20-26):
// out = (neg ? -1 : 1) * sum_k S[sx][k][a] * S[sy][k][b], k ascending.
struct ChainDesc {
    uint8_t sx, a, sy, b;
    uint16_t out;
    uint8_t neg, pad;
};

// Device layout of A ("panels"): the context's local rows are cut into panels
// of BR consecutive rows; panel q stores A(q*BR + r, k) at
// ((q * n) + k) * BR + r.  One k-row of a panel is BR contiguous doubles and a
// T x BR stage tile of the A.D kernel is one contiguous block (one bulk copy).
__host__ __device__ __forceinline__ size_t ap_idx(int n, int brs, int k, int il) {
    return ((static_cast<size_t>(il >> brs) * n + k) << brs) | static_cast<size_t>(il & ((1 << brs) - 1));
}

// Which device layout a context uses for A: exact contexts use the panel
// layout above; fast contexts use [r][kk] tiles (fast_kernels.cuh).
struct ALay {
    int fast;    // 0 panels (BR = 1 << brs), 1 fast tiles (64 x 36)
    int brs;
    int ntiles;  // fast: ceil(n / 36)
};
constexpr int kFastBRc = 64, kFastTc = 36;
__host__ __device__ __forceinline__ size_t a_idx(const ALay& L, int n, int k, int il) {
    if (!L.fast) return ap_idx(n, L.brs, k, il);
    const int q = il / kFastBRc, r = il % kFastBRc, t = k / kFastTc, kk = k % kFastTc;
    return ((static_cast<size_t>(q) * L.ntiles + t) * kFastBRc + r) * kFastTc + kk;
}
// storage index -> (k, il); the caller checks k < n and il < n_loc.
__host__ __device__ __forceinline__ void a_decode(const ALay& L, int n, size_t e, int& k, int& il) {
    if (!L.fast) {
        const int BR = 1 << L.brs;
        const size_t per = static_cast<size_t>(n) << L.brs;
        const size_t panel = e / per, rem = e - panel * per;
        k = static_cast<int>(rem >> L.brs);
        il = static_cast<int>(panel * BR + (rem & (BR - 1)));
    } else {
        const int kk = static_cast<int>(e % kFastTc);
        const size_t rest = e / kFastTc;
        const int r = static_cast<int>(rest % kFastBRc);
        const size_t rest2 = rest / kFastBRc;
        const int t = static_cast<int>(rest2 % L.ntiles);
        const size_t q = rest2 / L.ntiles;
        k = t * kFastTc + kk;
        il = static_cast<int>(q * kFastBRc + r);
    }
}

// Programmatic dependent launch (coopcg_gpu.cu pdl_launch): a kernel
// launched with programmatic stream serialization may be scheduled while the
// previous kernel in the stream drains; griddepcontrol.wait blocks until that
// kernel has completed and its memory is visible.  Every kernel of the
// iteration loop calls it before reading anything (a no-op otherwise).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next kernel of the stream be scheduled now (each CTA of this grid
// triggers; the dependent grid launches once all have).  Called by the
// fast-mode iteration-tail kernels, right after their own wait, so the next
// A.D can request its first A tiles (A is read-only during a solve) while the
// tail runs; the dependent still waits in griddepcontrol.wait for the rest.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- mbarrier + bulk async copy (TMA 1-D) helpers --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// One arrive per warp from lane 0, predicated instead of branched: a
// `if (lane == 0)` branch makes ptxas treat the code after it as divergent,
// which (for the chain kernel) costs the uniform loop and its schedule.
__device__ __forceinline__ void mbar_arrive_lane0(uint64_t* bar, int lane) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "setp.eq.s32 P1, %1, 0;\n"
        "@P1 mbarrier.arrive.shared::cta.b64 _, [%0];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(lane)
        : "memory");
}
// Global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// The same copy with an L2 evict-first policy: for A, streamed once per
// iteration (2.1-137 GB), so it does not push the small n x P blocks and
// partial sums that the other kernels of the iteration re-read out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// L2 residency across iterations ("A in L2"): the k-range of A
// below the context's res_k is copied with an evict-last policy, so that part of
// A (the same k-rows of every panel: every CTA reads the same share from L2)
// stays in L2 from one iteration's A.D to the next; the rest streams
// evict-first past it.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                     uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Fixed-order reduction of per-CTA partial vectors inside one CTA:
//   out[o] = sum_b part[b * stride + off + o * ostride],  o < nout.
// lpp threads per output each sum a strided subset with 8 independent loads in
// flight, then the lpp sub-sums are added in a fixed order (deterministic).
// `red` needs blockDim.x doubles of shared memory; all threads must call.
__device__ inline void cta_reduce_fixed(const double* __restrict__ part, int nparts, size_t stride, int off,
                                        int ostride, int nout, double* out, double* red) {
    const int nt = blockDim.x, tid = threadIdx.x;
    int lpp = nt / (nout > 0 ? nout : 1);
    lpp = lpp < 1 ? 1 : (lpp > 32 ? 32 : lpp);
    const int per_pass = nt / lpp;
    for (int base = 0; base < nout; base += per_pass) {
        const int o = base + tid / lpp, sub = tid % lpp;
        double s = 0.0;
        if (tid / lpp < per_pass && o < nout) {
            const double* src = part + off + static_cast<size_t>(o) * ostride;
            int b = sub;
            for (; b + 7 * lpp < nparts; b += 8 * lpp) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = src[static_cast<size_t>(b + u * lpp) * stride];
#pragma unroll
                for (int u = 0; u < 8; ++u) s += v[u];
            }
            for (; b < nparts; b += lpp) s += src[static_cast<size_t>(b) * stride];
        }
        red[tid] = s;
        __syncthreads();
        if (tid < per_pass && base + tid < nout) {
            double t = 0.0;
            for (int j = 0; j < lpp; ++j) t += red[tid * lpp + j];
            out[base + tid] = t;
        }
        __syncthreads();
    }
}

// Exact reference arithmetic: one rounding per operation, no contraction.
__device__ __forceinline__ double mac_exact(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}
__device__ __forceinline__ double msub_exact(double acc, double a, double b) {
    return __dsub_rn(acc, __dmul_rn(a, b));
}

} // namespace coopcg_gpu
