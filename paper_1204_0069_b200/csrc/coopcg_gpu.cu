// coopcg_gpu.cu -- host driver + C ABI of the B200-native cCG hot path.
//
// The driver reproduces the reference's drive() loop (coopcg/solvers.hpp:
// 259-283) on one CUDA stream: setup (stage_setup + setup_coordinator),
// then per iteration
//   ad_exact (Q = A D) -> chains (D^T Q, -R^T D, |D|^2) -> alpha_update
//   (alpha solve; R, X | X then R = A X - b) -> chains (-R^T Q, |R|^2) ->
//   beta_direction (beta solve + record + convergence; Dn = R + D beta^T,
//   Gram partials) -> rank_end (certificate / exact MGS, status, k++)
// and finalize_trace.  The coordinator decisions live on the device (Ctl):
// once a stop condition is reached every later kernel is a no-op, so the host
// enqueues iterations in chunks and only reads a small control snapshot per
// chunk (no per-iteration host round trip).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <type_traits>
#include <utility>

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed on first use (nccl_api)

#include "../../include/coopcg_gpu.h"
#include "common.cuh"
#include "exact_kernels.cuh"
#include "gen_kernels.cuh"
#include "fast_kernels.cuh"
#include "verify_kernels.cuh"

using namespace coopcg_gpu;

namespace coopcg_gpu {
// refgen.cu: the reference's random_spd (problem.hpp:118-152) on the device
int refgen_random_spd(double* At, ALay L, size_t ap_elems, int n, double cond, uint64_t seed, cudaStream_t st,
                      std::string& msg);
}  // namespace coopcg_gpu

namespace {

// A.D ring shape (rows of k per stage x stages), tools/probe/ad_probe.cu at the
// BASELINE sizes: 64 x 2 for P >= 8 (P=8: 0.420 vs 0.427 ms at n=16384; P=16:
// 8.87 vs 9.34 ms at n=65536; P=32: 66.5 vs 67.9 ms at n=131072), 32 x 4 at P=4.
template <int P>
constexpr int ad_T() { return P >= 8 ? 64 : 32; }
template <int P>
constexpr int ad_S() { return P >= 8 ? 2 : 4; }
constexpr int kChunkMax = 16;
constexpr int kMaxParts = 296;  // cap on per-CTA partial slots (2 x 148 SMs on a B200)
constexpr int kMaxDevices = 64;

int grid_for(size_t elems, int block) {
    size_t g = (elems + block - 1) / block;
    return (int)std::min<size_t>(g, 148ull * 16);
}
int pad_cols(int p) {
    int P = 4;
    while (P < p) P *= 2;
    return P;
}

// NCCL, loaded on first use by a rank context (coopcg_gpu_create_rank): the
// copy already mapped into the process (torch's) if there is one, else the
// system's libnccl.so.2.  Single-process contexts never load it.  The loaded
// table is the library's only process-wide state (initialised once).
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string err;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.err = std::string("dlopen(libnccl.so.2): ") + (e ? e : "?");
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) {
                ok = false;
                api.err += std::string(api.err.empty() ? "" : "; ") + "missing " + name;
            }
        };
        sym(api.getUniqueId, "ncclGetUniqueId");
        sym(api.commInitRank, "ncclCommInitRank");
        sym(api.commDestroy, "ncclCommDestroy");
        sym(api.broadcast, "ncclBroadcast");
        sym(api.groupStart, "ncclGroupStart");
        sym(api.groupEnd, "ncclGroupEnd");
        sym(api.errorString, "ncclGetErrorString");
        if (!ok) api.getUniqueId = nullptr;
    });
    return api;
}

// Even row blocks for `parts` shards, rounded up to 64-row panels when every
// shard keeps rows (coopcg_row_split; identical on every rank).
void row_split(int n, int parts, int part, int* r0, int* r1) {
    int per = (n + parts - 1) / parts;
    const int aligned = (per + 63) / 64 * 64;
    if ((long long)aligned * (parts - 1) < n) per = aligned;
    *r0 = std::min(n, part * per);
    *r1 = std::min(n, *r0 + per);
}

struct AdConfig {
    int BR = 64;
    int CPT = 4;
};

}  // namespace

struct coopcg_gpu_ctx {
    int n = 0, p = 0, P = 0, device = 0, arith = 0;
    int sms = 148;  // multiprocessors of `device` (queried at creation)
    int row0 = 0, row1 = 0, n_loc = 0, brs = 6, npanels = 0;
    size_t ap_elems = 0;
    ALay lay{0, 6, 0};
    // fast mode work decomposition (ad_fast_kernel): units = panels x kchunks
    int f_kchunks = 1, f_tpc = 1, f_units = 0, f_grid = 0, f_rgrid = 0, f_ugrid = 0;
    int f_rp = 4;  // fast_iter_kernel's rows per thread (fast_iter_rp)
    double* qpart = nullptr;     // kchunks x n_loc x P
    double* gpart = nullptr;     // rgrid x 4 P^2 (row-pass Gram partials)
    double* npart = nullptr;     // ugrid x P (norm partials)
    double* dtiles = nullptr;    // the A.D operand re-laid out as [col][kk] k-tiles
    double* gfin = nullptr;      // fast_iter_kernel: the reduced Grams (4 P^2)
    unsigned long long* gbar = nullptr;  // fast_iter_kernel: grid barrier arrival counter (monotonic)
    // A in L2 across iterations (set_l2_residency): the A.D copies A's k-rows
    // below res_k (exact) / k-tiles below res_k (fast) with an evict-last policy
    int res_k = 0;
    size_t res_bytes = 0;
    int fused_k = -1;            // iteration whose solve + update ran inside fast_iter_kernel
    bool fuse_ok = false;        // fast_iter_kernel's f_ugrid CTAs fit on the device at once
    bool a_ready = false, inputs_ready = false;
    cudaStream_t stream = nullptr;
    std::string msg;

    double* At = nullptr;
    double* X = nullptr;
    double* X0 = nullptr;  // uploaded starting block; copied into X at every solve start
    double* R = nullptr;
    double* Dblk[2] = {nullptr, nullptr};
    double* Q = nullptr;
    // peer-memory Q push (coopcg_gpu_ipc_handles / coopcg_gpu_set_peers): Q is
    // double-buffered by iteration parity (Qalt) so that a rank already pushing
    // iteration k+1's rows never overwrites rows a slower rank still reads in k
    double* Qalt = nullptr;
    bool p2p = false;
    PeerRows peers[2] = {};          // [parity]
    std::vector<void*> ipc_opened;   // mapped peer buffers (closed on destroy)
    double* S = nullptr;
    double* V = nullptr;  // MGS working copy
    double* b = nullptr;
    double* small = nullptr;
    double* partials = nullptr;
    double* init_norms = nullptr;  // P + 1
    double* final_norms = nullptr; // P + 1
    Ctl* ctl = nullptr;
    Ctl* ctl_host = nullptr;  // pinned snapshots [2]
    double* minres_host = nullptr;  // pinned [2][kChunkMax]: the chunk's recorded minres (enqueue sizing)
    unsigned char* trace_host = nullptr;  // pinned staging of the trace copy-out (end_impl)
    size_t trace_host_bytes = 0;
    ChainDesc* descs = nullptr;
    int desc_off[4] = {0, 0, 0, 0};
    int desc_cnt[4] = {0, 0, 0, 0};
    double* tr_norms = nullptr;
    double* tr_minres = nullptr;
    unsigned long long* tr_wall = nullptr;
    int tr_capacity = 0;
    double* stage = nullptr;  // host<->device staging, n * P doubles
    size_t stage_elems = 0;
    // A's host transfers (set_A / get_A_rows): two pinned + two device slots,
    // allocated on first use, so host copies overlap the PCIe copies
    double* pin[2] = {nullptr, nullptr};
    double* dslot[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    size_t pin_elems = 0;

    // verification mode (SolveOptions::keep_history / x_star, trace.hpp:84-87;
    // coopcg_gpu_set_verification): history entries of three n x P blocks
    // (X, R, D; entry 0 after setup, entry k + 1 after iteration k) and one row
    // of per-agent A-norm errors per iteration
    bool ver_hist_on = false, ver_xs_on = false;
    double* ver_hist = nullptr;
    int ver_hist_cap = 0;      // entries allocated
    double *ver_xs = nullptr, *ver_E = nullptr, *ver_AE = nullptr, *ver_anorm = nullptr;
    int ver_anorm_cap = 0;     // rows allocated
    int* ver_flag = nullptr;   // a_norm's "negative beyond round-off" (dense_ops.hpp:190-191)
    int ver_iters = -1;        // iterations of the last verification run (-1: none)

    AdConfig ad;
    int nparts = 0;

    std::vector<cudaEvent_t> mv_ev;  // [2 * 2 * kChunkMax]
    cudaEvent_t ev_run0 = nullptr, ev_run1 = nullptr, ev_loop0 = nullptr, ev_loop1 = nullptr;
    cudaEvent_t ev_chunk[2] = {nullptr, nullptr};
    // rank_end off the critical path (run_impl only): it runs on `side`,
    // concurrently with the next iteration's A.D, and is joined before the
    // first kernel that reads what it writes (ctl->k / stop / nsq_d).
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool rank_async = false;   // set by run_impl for its loop
    bool join_pending = false;
    coopcg_timing timing{};
    long long launches = 0;  // kernels launched since the last run started
    int phase_mv = 0;        // phase API: A.D launches timed so far in this solve (<= kChunkMax)
    int max_iters = 0, every = 50;  // resolved SolveOptions of the current solve
    int p_orig = 0;                 // agents at creation (mccg restricts ctx->p during a solve)
    int algo = 0;                   // 0 ccg, 1 mccg for the current solve
    int host_err = 0;               // error raised by the host-side mccg logic
    std::string host_err_msg;
    std::vector<int> ids;           // original id of each active slot
    // Householder generation in steps (coopcg_gpu_gen_householder_*): factors,
    // the vector w (all n rows; this context writes its own) and t1, t2
    double *hh_V = nullptr, *hh_lam = nullptr, *hh_w = nullptr, *hh_t = nullptr;
    int hh_m = -1;
    // ---- multi-GPU ---------------------------------------
    // A group handle (coopcg_gpu_create_multi): one process drives the row
    // shards `shards` (one per listed device; a device may repeat).  The
    // handle owns no device memory of its own; every call is routed to the
    // shards and the run loop enqueues every shard's work from this thread.
    std::vector<coopcg_gpu_ctx*> shards;
    std::vector<cudaEvent_t> gev;   // one cross-stream barrier event per shard
    // A rank context (coopcg_gpu_create_rank): one process per GPU, the row
    // exchanges are NCCL collectives on this context's stream.
    void* nccl = nullptr;           // ncclComm_t
    int nranks = 1, rank = 0;
    // COOPCG_GUARD=1 (debug): every device buffer sits between two guard
    // regions filled with a byte pattern; run / destroy check them
    struct Guarded {
        void* user;
        size_t bytes;
        const char* name;
    };
    std::vector<Guarded> guards;
};

// ---- device allocations (optionally guarded) ------------------------------
// COOPCG_GUARD=1: each buffer gets kGuardBytes of 0xA5 before and after it;
// check_guards() reports the first region a kernel wrote into.  A stand-in
// for compute-sanitizer's memcheck, which the GPU pool does not allow.
constexpr size_t kGuardBytes = 16384;
constexpr unsigned char kGuardByte = 0xA5;
static bool guard_enabled() {
    static const bool on = std::getenv("COOPCG_GUARD") != nullptr && std::getenv("COOPCG_GUARD")[0] == '1';
    return on;
}
template <typename T>
static cudaError_t gmalloc(coopcg_gpu_ctx* ctx, T** p, size_t bytes, const char* name) {
    if (!guard_enabled()) return cudaMalloc(reinterpret_cast<void**>(p), bytes);
    char* base = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuardBytes);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemset(base, kGuardByte, kGuardBytes)) != cudaSuccess) return e;
    if ((e = cudaMemset(base + kGuardBytes + bytes, kGuardByte, kGuardBytes)) != cudaSuccess) return e;
    *p = reinterpret_cast<T*>(base + kGuardBytes);
    ctx->guards.push_back({base + kGuardBytes, bytes, name});
    return cudaSuccess;
}
static void gfree(coopcg_gpu_ctx* ctx, void* p) {
    if (!p) return;
    if (guard_enabled()) {
        for (size_t i = 0; i < ctx->guards.size(); ++i)
            if (ctx->guards[i].user == p) {
                ctx->guards.erase(ctx->guards.begin() + i);
                cudaFree(static_cast<char*>(p) - kGuardBytes);
                return;
            }
    }
    cudaFree(p);
}
// 0, or 1 with `what` naming the first overwritten guard region.
static int check_guards(const coopcg_gpu_ctx* ctx, std::string& what) {
    std::vector<unsigned char> buf(kGuardBytes);
    for (const auto& g : ctx->guards)
        for (int side = 0; side < 2; ++side) {
            const char* at = side ? static_cast<const char*>(g.user) + g.bytes
                                  : static_cast<const char*>(g.user) - kGuardBytes;
            if (cudaMemcpy(buf.data(), at, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
                what = std::string("cannot read the guard of ") + g.name;
                return 1;
            }
            for (size_t i = 0; i < kGuardBytes; ++i)
                if (buf[i] != kGuardByte) {
                    char m[160];
                    std::snprintf(m, sizeof m, "device buffer %s: guard %s the buffer overwritten at byte %zu",
                                  g.name, side ? "after" : "before", i);
                    what = m;
                    return 1;
                }
        }
    return 0;
}

static void pin_give(double* p, size_t elems);  // the pinned staging cache (below)

static void hh_free(coopcg_gpu_ctx* ctx) {
    gfree(ctx, ctx->hh_V);
    gfree(ctx, ctx->hh_lam);
    gfree(ctx, ctx->hh_w);
    gfree(ctx, ctx->hh_t);
    ctx->hh_V = ctx->hh_lam = ctx->hh_w = ctx->hh_t = nullptr;
    ctx->hh_m = -1;
}

namespace {

thread_local std::string g_create_error;  // last coopcg_gpu_create* failure (ctx == NULL)

int fail(coopcg_gpu_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->msg = buf;
    else g_create_error = buf;
    return code;
}

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(ctx, COOPCG_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                     \
    } while (0)

#define CKL()                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                    \
        if (e_ != cudaSuccess)                                                                  \
            return fail(ctx, COOPCG_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                    \
    } while (0)

// ---- programmatic dependent launch ------------------------------------------
// Iteration-loop kernels are launched with programmatic stream serialization:
// the launch and CTA scheduling of kernel k+1 overlap the tail of kernel k,
// and kernel k+1's first statement (pdl_wait, griddepcontrol.wait) holds it
// until kernel k has completed.  COOPCG_NO_PDL=1 disables (A/B timing).
static bool pdl_enabled() {
    static const bool on = std::getenv("COOPCG_NO_PDL") == nullptr;
    return on;
}
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- A.D launcher: template dispatch on (P, CPT, BR) -------------------------
template <int P, int CPT, int BR>
size_t ad_smem() {
    return static_cast<size_t>(ad_S<P>()) * ad_T<P>() * (BR + P) * sizeof(double) + 2 * ad_S<P>() * sizeof(uint64_t);
}

// rows per thread: 2 at P >= 16 (one LDS.128 of A feeds 2 x CPT chains;
// tools/probe/ad_probe.cu: -11% / -12% time at P = 16 / 32), 1 otherwise.
template <int P>
constexpr int ad_rpt() { return P >= 16 ? 2 : 1; }
// the pipelined kernel (ad_exact_pipe_kernel) at P = 8 / BR = 128 and
// P = 16 / BR = 64 (panel heights pick_ad_config chooses for large n): 2 rows
// x 4 columns per thread, 64-row tiles, 3 stages; at P = 4 / BR = 32 (small
// n): 1 row x 2 columns, 128-row tiles, 4 stages (tools/probe/ad_v3_probe.cu)
template <int P, int BR>
constexpr bool ad_pipe() { return (P == 8 && BR == 128) || (P == 16 && BR == 64) || (P == 4 && BR == 32); }
template <int P>
constexpr int pipe_T() { return P == 4 ? 128 : 64; }
template <int P>
constexpr int pipe_S() { return P == 4 ? 4 : 3; }
template <int P>
constexpr int pipe_CPT() { return P == 4 ? 2 : 4; }
template <int P>
constexpr int pipe_RPT() { return P == 4 ? 1 : 2; }

template <int P, int CPT, int BR>
cudaError_t ad_launch_t(coopcg_gpu_ctx* ctx, const double* src, double* dst, const double* b, const int* stop,
                        const PeerRows& peers) {
    constexpr bool pipe = ad_pipe<P, BR>();
    constexpr int RPT = pipe ? pipe_RPT<P>() : ad_rpt<P>();
    constexpr int KC = pipe ? pipe_CPT<P>() : CPT;  // columns per thread of the chosen kernel
    constexpr int PT = pipe_T<P>(), PS = pipe_S<P>();
    constexpr int T = ad_T<P>(), S = ad_S<P>();
    const bool push = peers.n > 0;
    using Kern = void (*)(const double*, int, int, int, const double*, double*, const double*, int, const int*,
                          PeerRows, int);
    Kern kern;
    if constexpr (pipe)
        kern = push ? ad_exact_pipe_kernel<P, KC, RPT, BR, PT, PS, true>
                    : ad_exact_pipe_kernel<P, KC, RPT, BR, PT, PS, false>;
    else if constexpr (RPT == 1)
        kern = push ? ad_exact_kernel<P, CPT, BR, T, S, true> : ad_exact_kernel<P, CPT, BR, T, S, false>;
    else
        kern = push ? ad_exact_rpt_kernel<P, CPT, BR, T, S, 2, true> : ad_exact_rpt_kernel<P, CPT, BR, T, S, 2, false>;
    const size_t smem = pipe ? ad_pipe_smem(P, BR, PT, PS) : ad_smem<P, CPT, BR>();
    // the shared-memory opt-in, once per (instantiation, device); thread-safe
    static std::once_flag attr_once[2][kMaxDevices];
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[push][ctx->device % kMaxDevices], [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return attr_err;
    dim3 grid((ctx->n_loc + BR - 1) / BR);
    dim3 block(32 + 32 * ad_consumer_warps(BR / RPT, P / KC));
    pdl_launch(kern, dim3(grid), dim3(block), smem, ctx->stream, ctx->At, ctx->n, ctx->n_loc, ctx->row0, src, dst, b, ctx->p, stop,
               peers, ctx->res_k);
    ++ctx->launches;
    return cudaGetLastError();
}

template <int P, int CPT>
cudaError_t ad_launch_br(coopcg_gpu_ctx* ctx, const double* src, double* dst, const double* b, const int* stop,
                         const PeerRows& peers) {
    switch (ctx->ad.BR) {
    case 32: return ad_launch_t<P, CPT, 32>(ctx, src, dst, b, stop, peers);
    case 128:
        if constexpr (P == 8) return ad_launch_t<P, CPT, 128>(ctx, src, dst, b, stop, peers);
        return cudaErrorInvalidValue;
    default: return ad_launch_t<P, CPT, 64>(ctx, src, dst, b, stop, peers);
    }
}

// peers: push the rows to every rank's copy of dst (row-sharded Q, peer mode)
cudaError_t ad_launch(coopcg_gpu_ctx* ctx, const double* src, double* dst, const double* b, const int* stop,
                      const PeerRows& peers = PeerRows{}) {
    switch (ctx->P) {
    case 4: return ad_launch_br<4, 2>(ctx, src, dst, b, stop, peers);
    case 8: return ad_launch_br<8, 4>(ctx, src, dst, b, stop, peers);
    case 16: return ad_launch_br<16, 4>(ctx, src, dst, b, stop, peers);
    default: return ad_launch_br<32, 4>(ctx, src, dst, b, stop, peers);
    }
}

// ---- fast-mode launchers ------------------------------------------------------
template <int P>
size_t fast_ad_smem() {
    return (size_t)fast_stages<P>() * (kFastBR * kFastT + kFastT * P) * sizeof(double) +
           2 * fast_stages<P>() * sizeof(uint64_t);
}
// column groups per CTA: P=8 -> 1 (2 DMMA warps), P=16/32 -> 2 (4 DMMA warps)
template <int P>
constexpr int fast_wn() { return P >= 16 ? 2 : 1; }
// M-tiles (8 rows) per consumer warp.  P >= 16: 4 (WN = 2 already gives four DMMA
// warps per CTA).  P = 8: 2 when A is small (four DMMA warps per CTA: one warp issues a DMMA
// only every ~32 cycles, and a launch of a few tens of microseconds is bound by that issue
// rate, not by HBM -- cfg 1 A.D 29.4 -> 28.1 us), 4 when A streams from HBM for hundreds of
// microseconds (cfg 2: 315 vs 327 us; fewer warps, less power under sw_power_cap).  The
// results are bit-identical for any MT (each element's k order is unchanged).
// The build macro COOPCG_FAST_MT8 = 2 / 4 or the environment variable
// COOPCG_FAST_MT = 2 / 4 force one shape.
constexpr size_t kFastSmallA = (size_t)1 << 26;  // elements of the local A block
template <int P, int MT>
cudaError_t fast_ad_mt(coopcg_gpu_ctx* ctx, const double* src, const int* stop) {
    constexpr int WN = fast_wn<P>();
    constexpr bool TR = P >= 16;
    auto kern = ad_fast_kernel<P, WN, TR, MT>;
    static std::once_flag attr_once[kMaxDevices];
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[ctx->device % kMaxDevices], [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_ad_smem<P>());
    });
    if (attr_err != cudaSuccess) return attr_err;
    const double* operand = src;
    if (TR) {  // operand -> [col][kk] k-tiles (conflict-free B fragments at P >= 16)
        const size_t tot = (size_t)ctx->lay.ntiles * P * kFastT;
        pdl_launch(operand_tiles_kernel<P>, dim3(grid_for(tot, 256)), dim3(256), 0, ctx->stream, src, ctx->n, ctx->lay.ntiles,
                                                                             ctx->dtiles, stop);
        ++ctx->launches;
        operand = ctx->dtiles;
    }
    pdl_launch(kern, dim3(ctx->f_grid), dim3(32 + 32 * (kFastBR / (8 * MT)) * WN), fast_ad_smem<P>(), ctx->stream, 
        ctx->At, ctx->n, ctx->n_loc, ctx->lay.ntiles, operand, ctx->qpart, ctx->f_kchunks, ctx->f_tpc,
        ctx->f_units, stop, ctx->res_k);
    ++ctx->launches;
    return cudaGetLastError();
}
template <int P>
cudaError_t fast_ad_t(coopcg_gpu_ctx* ctx, const double* src, const int* stop) {
    if constexpr (P == 8) {
#ifdef COOPCG_FAST_MT8
        return fast_ad_mt<8, COOPCG_FAST_MT8>(ctx, src, stop);
#else
        static const int mt_env = [] {
            const char* e = std::getenv("COOPCG_FAST_MT");
            return e ? std::atoi(e) : 0;
        }();
        const bool small = mt_env == 2 || (mt_env != 4 && (size_t)ctx->n_loc * ctx->n <= kFastSmallA);
        if (small) return fast_ad_mt<8, 2>(ctx, src, stop);
        return fast_ad_mt<8, 4>(ctx, src, stop);
#endif
    } else {
        return fast_ad_mt<P, 4>(ctx, src, stop);
    }
}
cudaError_t fast_ad(coopcg_gpu_ctx* ctx, const double* src, const int* stop) {
    switch (ctx->P) {
    case 8: return fast_ad_t<8>(ctx, src, stop);
    case 16: return fast_ad_t<16>(ctx, src, stop);
    default: return fast_ad_t<32>(ctx, src, stop);
    }
}
template <int P>
cudaError_t fast_rows_t(coopcg_gpu_ctx* ctx, double* dst, const double* b, const double* D, const double* R,
                        const double* Qfull, int mode, const int* stop, const PeerRows& peers) {
    ++ctx->launches;
    auto kern = peers.n > 0 ? fast_rows_kernel<P, true> : fast_rows_kernel<P, false>;
    return pdl_launch(kern, dim3(ctx->f_rgrid), dim3(256), 0, ctx->stream, ctx->qpart, ctx->f_kchunks, ctx->n_loc,
                      ctx->row0, dst, b, D, R, Qfull, ctx->p, mode, ctx->gpart, stop, peers);
}
cudaError_t fast_rows(coopcg_gpu_ctx* ctx, double* dst, const double* b, const double* D, const double* R,
                      const double* Qfull, int mode, const int* stop, const PeerRows& peers = PeerRows{}) {
    switch (ctx->P) {
    case 8: return fast_rows_t<8>(ctx, dst, b, D, R, Qfull, mode, stop, peers);
    case 16: return fast_rows_t<16>(ctx, dst, b, D, R, Qfull, mode, stop, peers);
    default: return fast_rows_t<32>(ctx, dst, b, D, R, Qfull, mode, stop, peers);
    }
}
template <int P>
cudaError_t fast_update_t(coopcg_gpu_ctx* ctx, const double* Q, const double* D, double* Dn, int mode, const int* stop) {
    pdl_launch(fast_update_kernel<P>, dim3(ctx->f_ugrid), dim3(256), 0, ctx->stream, ctx->X, ctx->R, Q, D, Dn, ctx->small, ctx->n,
                                                                 ctx->p, mode, ctx->npart, ctx->partials, stop);
    ++ctx->launches;
    return cudaGetLastError();
}
cudaError_t fast_update(coopcg_gpu_ctx* ctx, const double* Q, const double* D, double* Dn, int mode,
                        const int* stop) {
    switch (ctx->P) {
    case 8: return fast_update_t<8>(ctx, Q, D, Dn, mode, stop);
    case 16: return fast_update_t<16>(ctx, Q, D, Dn, mode, stop);
    default: return fast_update_t<32>(ctx, Q, D, Dn, mode, stop);
    }
}
template <int P>
cudaError_t fast_solve_t(coopcg_gpu_ctx* ctx, int mode) {
    // flat Grams + the reduction scratch (+ solve_cta's five P x (P+1) buffers at P >= 16)
    const size_t smem = (size_t)(4 * P * P + 1024 + (P >= COOPCG_CTA_SOLVE_MIN_P ? 5 * P * (P + 1) : 0)) * sizeof(double);
    static std::once_flag attr_once[kMaxDevices];
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[ctx->device % kMaxDevices], [&] {
        attr_err = cudaFuncSetAttribute(fast_solve_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return attr_err;
    return pdl_launch(fast_solve_kernel<P>, dim3(1), dim3(1024), smem, ctx->stream, ctx->gpart, ctx->f_rgrid, ctx->small,
                      ctx->ctl, mode);
}
cudaError_t fast_solve(coopcg_gpu_ctx* ctx, int mode) {
    ++ctx->launches;
    switch (ctx->P) {
    case 4: return fast_solve_t<4>(ctx, mode);
    case 8: return fast_solve_t<8>(ctx, mode);
    case 16: return fast_solve_t<16>(ctx, mode);
    default: return fast_solve_t<32>(ctx, mode);
    }
}

// The fused post-MMA iteration (fast_iter_kernel): one cooperative launch of
// f_ugrid CTAs (== f_rgrid on an unsharded context), all co-resident.
// COOPCG_NO_FUSE=1 runs the separate row / solve / update kernels instead.
static bool fuse_enabled() {
    static const bool on = std::getenv("COOPCG_NO_FUSE") == nullptr;
    return on;
}
template <int P, int RP>
cudaError_t fast_iter_t(coopcg_gpu_ctx* ctx, double* Q, const double* D, double* Dn) {
    auto kern = fast_iter_kernel<P, RP>;
    const size_t smem = fused_smem_bytes<P, RP>();
    static std::once_flag attr_once[kMaxDevices];
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[ctx->device % kMaxDevices], [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctx->f_ugrid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    ++ctx->launches;
    return cudaLaunchKernelEx(&cfg, kern, (const double*)ctx->qpart, ctx->f_kchunks, ctx->n, Q, ctx->X, ctx->R, D, Dn,
                              ctx->small, ctx->ctl, ctx->p, ctx->gpart, ctx->gfin, ctx->npart, ctx->partials,
                              ctx->gbar);
}
template <int P, int RP>
bool fast_iter_fits_t(const coopcg_gpu_ctx* ctx) {
    int occ = 0;
    if (cudaFuncSetAttribute(fast_iter_kernel<P, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)fused_smem_bytes<P, RP>()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fast_iter_kernel<P, RP>, 256, fused_smem_bytes<P, RP>()) !=
            cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return occ * ctx->sms >= ctx->f_ugrid && ctx->f_ugrid == ctx->f_rgrid;
}
template <int P>
bool fast_iter_fits_p(const coopcg_gpu_ctx* ctx) {
    switch (ctx->f_rp) {
    case 1: return fast_iter_fits_t<P, 1>(ctx);
    case 2: return fast_iter_fits_t<P, 2>(ctx);
    default: return fast_iter_fits_t<P, 4>(ctx);
    }
}
bool fast_iter_fits(const coopcg_gpu_ctx* ctx) {
    switch (ctx->P) {
    case 8: return fast_iter_fits_p<8>(ctx);
    case 16: return fast_iter_fits_p<16>(ctx);
    default: return fast_iter_fits_p<32>(ctx);
    }
}
template <int P>
cudaError_t fast_iter_p(coopcg_gpu_ctx* ctx, double* Q, const double* D, double* Dn) {
    switch (ctx->f_rp) {
    case 1: return fast_iter_t<P, 1>(ctx, Q, D, Dn);
    case 2: return fast_iter_t<P, 2>(ctx, Q, D, Dn);
    default: return fast_iter_t<P, 4>(ctx, Q, D, Dn);
    }
}
cudaError_t fast_iter(coopcg_gpu_ctx* ctx, double* Q, const double* D, double* Dn) {
    switch (ctx->P) {
    case 8: return fast_iter_p<8>(ctx, Q, D, Dn);
    case 16: return fast_iter_p<16>(ctx, Q, D, Dn);
    default: return fast_iter_p<32>(ctx, Q, D, Dn);
    }
}

AdConfig pick_ad_config(int n_loc, int P, int sms) {
    AdConfig c;
    // Measured sweep (tools/probe/ad_probe.cu, profiles/; ring shapes: ad_T / ad_S);
    // P=4: 2 cols/thread (7.1 TB/s at n=16384), P=8: 4 (5.0 TB/s),
    // P=16/32: 4 cols x 2 rows (FP64-issue bound in exact mode, ~13 of 18 T instr/s).
    // Above one CTA per SM at BR = 64, P = 8 switches to 128-row panels for the
    // pipelined kernel (tools/probe/ad_v3_probe.cu).
    c.BR = (n_loc >= sms * 64) ? 64 : 32;
    if (P == 8 && n_loc > sms * 64) c.BR = 128;
    c.CPT = (P == 4) ? 2 : 4;  // with 2 rows per thread at P >= 16
    return c;
}

// ---- A in L2 across iterations ------------------------------------------------
// A is re-read by every iteration's A.D; the part of it that fits next to the
// iteration's other working set (the n x P blocks, the k-chunk partials) can
// stay in the 126 MB L2 from one iteration to the next.  The resident part is
// the first res_k k-rows of every panel (exact) or the first res_k k-tiles of
// every (panel, k-chunk) work unit (fast), so every A.D CTA reads the same
// share of its stream from L2 and the HBM part is spread over all CTAs.
// Budget: COOPCG_L2_RES_MB (0 disables), split among the contexts sharing a
// device (`share`).
// Default (no COOPCG_L2_RES_MB): fast mode keeps half of L2 for A when the local
// A block is larger than ~3/4 of L2 (below that all of A stays in L2 anyway) and
// at most 1 GB (above, the resident share is a few percent of the stream: cfg 2
// +-1%).  cfg 1 (134 MB, round 2 session 4, tools/l2res_fast.sh): A.D 28.1 us at
// 0 MB, 24.6 at 64 MB, 24.1 at 80 MB, 28.0 at 112 MB; 25.8k -> 27.1k it/s at
// 64 MB (the iteration tail wants its own share of L2).  The exact mode's
// small-n A.D is FP64-issue bound, not HBM bound: off unless asked for.
double l2_res_budget_mb(const coopcg_gpu_ctx* ctx) {
    static const double env_mb = [] {
        const char* e = std::getenv("COOPCG_L2_RES_MB");
        return e ? std::max(0.0, std::atof(e)) : -1.0;
    }();
    if (env_mb >= 0.0) return env_mb;
    if (ctx->arith != COOPCG_ARITH_FAST) return 0.0;
    int l2 = 0;
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess || l2 <= 0) return 0.0;
    const double a_bytes = (double)ctx->n_loc * ctx->n * 8.0;
    if (a_bytes < 0.75 * l2 || a_bytes > 1e9) return 0.0;
    return 0.5 * l2 / 1e6;
}
void set_l2_residency(coopcg_gpu_ctx* ctx, int share) {
    const double budget = l2_res_budget_mb(ctx) * 1e6 / std::max(1, share);
    // bytes of A per unit of res_k: one k-row of every panel (exact) or one
    // k-tile of every (panel, k-chunk) work unit (fast: the first res_k tiles
    // of EVERY unit, so each CTA reads the same share from L2 and the HBM part
    // is spread over all CTAs -- a CTA's stream is bound by its ring depth)
    const double unit = ctx->arith == COOPCG_ARITH_FAST
                            ? (double)ctx->npanels * ctx->f_kchunks * kFastBR * kFastT * 8.0
                            : (double)ctx->npanels * ctx->ad.BR * 8.0;
    const int units = ctx->arith == COOPCG_ARITH_FAST ? ctx->f_tpc : ctx->n;
    ctx->res_k = (int)std::min<double>(units, std::floor(budget / unit));
    ctx->res_bytes = (size_t)(ctx->res_k * unit);
}

// ---- the p x p solves fused into their elementwise consumers ----------------
// Every CTA redoes the solve, so the grid must fit in one wave: one CTA per
// step of kUpdTiles x 256 elements, at most (resident CTAs per SM) x SMs, and
// for the direction pass at most nparts (the certificate sums one Gram
// partial per CTA).
template <typename K>
int one_wave(K kern, int cap) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    return std::max(1, std::min(cap, std::max(occ, 1) * sms));
}
static int blocks_of(int n, int P) { return (n * P + kUpdTiles * 256 - 1) / (kUpdTiles * 256); }

template <int P>
cudaError_t alpha_update_launch_t(coopcg_gpu_ctx* ctx, const double* Q, const double* D, int mode) {
    static const int wave = one_wave(alpha_update_kernel<P>, 1 << 30);
    const int grid = std::min(wave, blocks_of(ctx->n, P));
    return pdl_launch(alpha_update_kernel<P>, dim3(grid), dim3(256), 0, ctx->stream, ctx->R, ctx->X, Q, D, ctx->small,
                      ctx->n, ctx->p, mode, ctx->ctl);
}
template <int P>
int beta_direction_grid_t(const coopcg_gpu_ctx* ctx) {
    static const int wave = one_wave(beta_direction_kernel<P>, kMaxParts);
    return std::min({wave, ctx->nparts, blocks_of(ctx->n, P)});
}
template <int P>
cudaError_t beta_direction_launch_t(coopcg_gpu_ctx* ctx, const double* D, double* Dn) {
    return pdl_launch(beta_direction_kernel<P>, dim3(beta_direction_grid_t<P>(ctx)), dim3(256), 0, ctx->stream, ctx->R,
                      D, Dn, ctx->small, ctx->n, ctx->p, ctx->partials, ctx->ctl, ctx->tr_norms, ctx->tr_minres,
                      ctx->tr_wall, ctx->tr_capacity, ctx->algo == 2 ? 1 : 0);
}
// alpha solve + X (and R) update, iteration mode 0 (recurrence) / 1 (recompute)
cudaError_t alpha_update_launch(coopcg_gpu_ctx* ctx, const double* Q, const double* D, int mode) {
    ++ctx->launches;
    switch (ctx->P) {
    case 4: return alpha_update_launch_t<4>(ctx, Q, D, mode);
    case 8: return alpha_update_launch_t<8>(ctx, Q, D, mode);
    case 16: return alpha_update_launch_t<16>(ctx, Q, D, mode);
    default: return alpha_update_launch_t<32>(ctx, Q, D, mode);
    }
}
// beta solve + record + convergence, then Dn = R + D beta^T with Gram partials
cudaError_t beta_direction_launch(coopcg_gpu_ctx* ctx, const double* D, double* Dn) {
    ++ctx->launches;
    switch (ctx->P) {
    case 4: return beta_direction_launch_t<4>(ctx, D, Dn);
    case 8: return beta_direction_launch_t<8>(ctx, D, Dn);
    case 16: return beta_direction_launch_t<16>(ctx, D, Dn);
    default: return beta_direction_launch_t<32>(ctx, D, Dn);
    }
}
// Exact-mode count of Gram partials (= the direction pass's grid).
int exact_dgrid(const coopcg_gpu_ctx* ctx) {
    switch (ctx->P) {
    case 4: return beta_direction_grid_t<4>(ctx);
    case 8: return beta_direction_grid_t<8>(ctx);
    case 16: return beta_direction_grid_t<16>(ctx);
    default: return beta_direction_grid_t<32>(ctx);
    }
}
// Gram partials of an existing block D (setup D0, the rank entry point).
cudaError_t gram_partials_launch(coopcg_gpu_ctx* ctx, const double* D, int grid, const int* stop) {
    const int n = ctx->n, p = ctx->p;
    switch (ctx->P) {
    case 4: gram_partials_kernel<4><<<grid, 256, 0, ctx->stream>>>(D, n, p, ctx->partials, stop); break;
    case 8: gram_partials_kernel<8><<<grid, 256, 0, ctx->stream>>>(D, n, p, ctx->partials, stop); break;
    case 16: gram_partials_kernel<16><<<grid, 256, 0, ctx->stream>>>(D, n, p, ctx->partials, stop); break;
    default: gram_partials_kernel<32><<<grid, 256, 0, ctx->stream>>>(D, n, p, ctx->partials, stop); break;
    }
    return cudaGetLastError();
}

// ---- chain launcher ---------------------------------------------------------
enum ChainPhase { kPhSetup = 0, kPhGram = 1, kPhBeta = 2, kPhFinal = 3 };

// NSRC_MAX: the most sources any launch of this instantiation streams
template <int P, int T, int S, int NSRC_MAX = 3>
cudaError_t chains_launch_t(coopcg_gpu_ctx* ctx, int phase, const double* s0, const double* s1, const double* s2,
                            int nsrc, const int* stop) {
    auto kern = chain_kernel<P, T, S>;
    const size_t smem_max = chain_smem_bytes(P, T, S, NSRC_MAX);
    static std::once_flag attr_once[kMaxDevices];
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[ctx->device % kMaxDevices], [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    });
    if (attr_err != cudaSuccess) return attr_err;
    const int cnt = ctx->desc_cnt[phase];
    const size_t smem = chain_smem_bytes(P, T, S, nsrc);
    pdl_launch(kern, dim3((cnt + 63) / 64), dim3(kChainThreads), smem, ctx->stream, s0, s1, s2, nsrc, ctx->n, ctx->descs + ctx->desc_off[phase],
                                                     cnt, ctx->small, stop);
    ++ctx->launches;
    return cudaGetLastError();
}

// Rings (tools/probe/chain_kernel_probe.cu, n = 16384): 3 stages of the
// longest tile that fits (per-tile overhead dominates shorter tiles):
// P=4: 512 rows (93 us per phase vs 99 at 256); P=8: 384 with three sources
// (96.5 vs 98.6), 512 with at most two (the beta / setup / final phases);
// P=16: 192 (105 vs 115 us at 4 x 128); P=32: 96 (127 vs 144 us at 4 x 64).
cudaError_t chains_launch(coopcg_gpu_ctx* ctx, int phase, const double* s0, const double* s1, const double* s2,
                          int nsrc, const int* stop) {
    switch (ctx->P) {
    case 4: return chains_launch_t<4, 512, 3>(ctx, phase, s0, s1, s2, nsrc, stop);
    case 8:
        return nsrc <= 2 ? chains_launch_t<8, 512, 3, 2>(ctx, phase, s0, s1, s2, nsrc, stop)
                         : chains_launch_t<8, 384, 3>(ctx, phase, s0, s1, s2, nsrc, stop);
    case 16: return chains_launch_t<16, 192, 3>(ctx, phase, s0, s1, s2, nsrc, stop);
    default: return chains_launch_t<32, 96, 3>(ctx, phase, s0, s1, s2, nsrc, stop);
    }
}

void build_descs(int p, int P, std::vector<ChainDesc>& all, int off[4], int cnt[4]) {
    const SmallLayout L{P};
    auto add = [&](int sx, int a, int sy, int b, int out, int neg) {
        ChainDesc d;
        d.sx = (uint8_t)sx;
        d.a = (uint8_t)a;
        d.sy = (uint8_t)sy;
        d.b = (uint8_t)b;
        d.out = (uint16_t)out;
        d.neg = (uint8_t)neg;
        d.pad = 0;
        all.push_back(d);
    };
    // setup: |R_i|^2 (stage_setup, block_cg.hpp:140)        srcs: 0=R
    off[kPhSetup] = (int)all.size();
    for (int i = 0; i < p; ++i) add(0, i, 0, i, L.nsq_r() + i, 0);
    cnt[kPhSetup] = (int)all.size() - off[kPhSetup];
    // gram: raw(i,j) = D_i.Q_j; rhs_a(i,j) = -R_i.D_j; |D_i|^2   srcs: 0=D 1=Q 2=R
    off[kPhGram] = (int)all.size();
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) add(0, i, 1, j, L.raw() + i * P + j, 0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) add(2, i, 0, j, L.rhs_a() + i * P + j, 1);
    for (int i = 0; i < p; ++i) add(0, i, 0, i, L.nsq_d() + i, 0);
    cnt[kPhGram] = (int)all.size() - off[kPhGram];
    // beta: rhs_b(i,j) = -R_i.Q_j; |R_i|^2                    srcs: 0=R 1=Q
    off[kPhBeta] = (int)all.size();
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) add(0, i, 1, j, L.rhs_b() + i * P + j, 1);
    for (int i = 0; i < p; ++i) add(0, i, 0, i, L.nsq_r() + i, 0);
    cnt[kPhBeta] = (int)all.size() - off[kPhBeta];
    // final: |A x_j - b|^2                                    srcs: 0=S
    off[kPhFinal] = (int)all.size();
    for (int i = 0; i < p; ++i) add(0, i, 0, i, L.nsq_f() + i, 0);
    cnt[kPhFinal] = (int)all.size() - off[kPhFinal];
}

size_t rank_smem(int P) { return 2ull * kRankTile * P * sizeof(double) + 2 * sizeof(uint64_t); }


int destroy_impl(coopcg_gpu_ctx* ctx) {
    if (!ctx) return COOPCG_OK;
#ifdef COOPCG_PHASE_TIMES
    {
        unsigned long long h[16] = {0};
        cudaSetDevice(ctx->device);
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_phase_ns, sizeof h);
        if (h[7])
            std::fprintf(stderr,
                         "fast_iter phases (CTA 0, mean over %llu): A %.2f  bar1 %.2f  B %.2f  bar2 %.2f  C-load %.2f  "
                         "C-solve %.2f  D %.2f us\n",
                         h[7], h[0] * 1e-3 / h[7], h[1] * 1e-3 / h[7], h[2] * 1e-3 / h[7], h[3] * 1e-3 / h[7],
                         h[4] * 1e-3 / h[7], h[5] * 1e-3 / h[7], h[6] * 1e-3 / h[7]);
        std::fprintf(stderr, "  C-solve: setup %.2f  cholesky %.2f  alpha %.2f  beta %.2f us\n", h[8] * 1e-3 / h[7],
                     h[9] * 1e-3 / h[7], h[10] * 1e-3 / h[7], h[11] * 1e-3 / h[7]);
        const unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase_ns, z, sizeof z);
    }
#endif
    for (size_t g = 0; g < ctx->gev.size(); ++g) {
        cudaSetDevice(ctx->shards[g]->device);
        if (ctx->gev[g]) cudaEventDestroy(ctx->gev[g]);
    }
    for (coopcg_gpu_ctx* c : ctx->shards) destroy_impl(c);
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->nccl) nccl_api().commDestroy(static_cast<ncclComm_t>(ctx->nccl));
    gfree(ctx, ctx->At);
    gfree(ctx, ctx->X);
    gfree(ctx, ctx->X0);
    gfree(ctx, ctx->R);
    gfree(ctx, ctx->Dblk[0]);
    gfree(ctx, ctx->Dblk[1]);
    for (void* ptr : ctx->ipc_opened) cudaIpcCloseMemHandle(ptr);
    gfree(ctx, ctx->Qalt);
    gfree(ctx, ctx->Q);
    gfree(ctx, ctx->S);
    gfree(ctx, ctx->V);
    gfree(ctx, ctx->b);
    gfree(ctx, ctx->qpart);
    gfree(ctx, ctx->gpart);
    hh_free(ctx);
    gfree(ctx, ctx->npart);
    gfree(ctx, ctx->dtiles);
    gfree(ctx, ctx->gfin);
    gfree(ctx, ctx->gbar);
    gfree(ctx, ctx->small);
    gfree(ctx, ctx->partials);
    gfree(ctx, ctx->init_norms);
    gfree(ctx, ctx->final_norms);
    gfree(ctx, ctx->ctl);
    gfree(ctx, ctx->descs);
    gfree(ctx, ctx->tr_norms);
    gfree(ctx, ctx->tr_minres);
    gfree(ctx, ctx->tr_wall);
    gfree(ctx, ctx->stage);
    gfree(ctx, ctx->ver_hist);
    gfree(ctx, ctx->ver_xs);
    gfree(ctx, ctx->ver_E);
    gfree(ctx, ctx->ver_AE);
    gfree(ctx, ctx->ver_anorm);
    gfree(ctx, ctx->ver_flag);
    for (int q = 0; q < 2; ++q) {
        pin_give(ctx->pin[q], ctx->pin_elems);
        gfree(ctx, ctx->dslot[q]);
        if (ctx->pin_ev[q]) cudaEventDestroy(ctx->pin_ev[q]);
    }
    if (ctx->ctl_host) cudaFreeHost(ctx->ctl_host);
    if (ctx->minres_host) cudaFreeHost(ctx->minres_host);
    if (ctx->trace_host) cudaFreeHost(ctx->trace_host);
    for (auto e : ctx->mv_ev) cudaEventDestroy(e);
    cudaEvent_t evs[] = {ctx->ev_run0,      ctx->ev_run1,      ctx->ev_loop0, ctx->ev_loop1,
                         ctx->ev_chunk[0], ctx->ev_chunk[1], ctx->ev_fork,  ctx->ev_join};
    for (auto e : evs)
        if (e) cudaEventDestroy(e);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return COOPCG_OK;
}

int ensure_trace_capacity(coopcg_gpu_ctx* ctx, int cap) {
    if (cap <= ctx->tr_capacity) return COOPCG_OK;
    gfree(ctx, ctx->tr_norms);
    gfree(ctx, ctx->tr_minres);
    gfree(ctx, ctx->tr_wall);
    ctx->tr_norms = nullptr;
    ctx->tr_minres = nullptr;
    ctx->tr_wall = nullptr;
    // rows are p_orig wide (the kernels write tr_norms[k * p0 + j]; a previous
    // mccg solve may have left ctx->p reduced)
    CK(gmalloc(ctx, &ctx->tr_norms, sizeof(double) * (size_t)cap * ctx->p_orig, "tr_norms"));
    CK(gmalloc(ctx, &ctx->tr_minres, sizeof(double) * (size_t)cap, "tr_minres"));
    CK(gmalloc(ctx, &ctx->tr_wall, sizeof(unsigned long long) * (size_t)cap, "tr_wall"));
    ctx->tr_capacity = cap;
    return COOPCG_OK;
}

// Host part of the generators, shared by the C ABI.
uint64_t host_draw(uint64_t key, uint64_t c) { return mix64(key + c * kGolden); }
double host_unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
double host_uniform_pm1(uint64_t key, uint64_t c) {
    volatile double u = host_unit(host_draw(key, c));
    volatile double t = 2.0 * u;
    return -1.0 + t;
}
double host_normal(uint64_t key, uint64_t t) {
    double u1 = host_unit(host_draw(key, 2 * t + 1));
    double u2 = host_unit(host_draw(key, 2 * t + 2));
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    volatile double l = -2.0 * std::log(u1);
    const double r = std::sqrt(l);
    const double two_pi = 6.283185307179586476925286766559;
    volatile double ang = two_pi * u2;
    volatile double cs = std::cos(ang);
    return r * cs;
}

}  // namespace

// memcpy on several host threads (a single core copies ~10 GB/s; the
// PCIe 5 link and host DRAM take several times that).
static unsigned copy_threads() {
    static const unsigned t = [] {
        const char* e = std::getenv("COOPCG_COPY_THREADS");
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        return e ? std::max(1u, (unsigned)std::atoi(e)) : std::min(16u, hw);
    }();
    return t;
}
static void par_memcpy(void* dst, const void* src, size_t bytes) {
    const unsigned T = bytes >= (size_t(4) << 20) ? copy_threads() : 1u;
    if (T <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = ((bytes + T - 1) / T + 4095) & ~size_t(4095);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) {
        const size_t o = t * per;
        if (o >= bytes) break;
        th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                                          std::min(per, bytes - o)); });
    }
    for (auto& x : th) x.join();
}

// Pinned host staging for A's transfers, cached process-wide: page-locking
// 2 x 32 MB costs ~70 ms, which a one-shot call (create, set_A, solve,
// destroy -- the drop-in ccg_solve) would otherwise pay every time.  A
// mutex-guarded free list of slot buffers (portable pinned memory, any
// device); contexts take one on first use and give it back on destroy.
struct PinCache {
    std::mutex mu;
    std::vector<std::pair<double*, size_t>> free;  // (buffer, elements)
};
static PinCache& pin_cache() {
    static PinCache c;
    return c;
}
static double* pin_take(size_t elems) {
    PinCache& c = pin_cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        for (size_t i = 0; i < c.free.size(); ++i)
            if (c.free[i].second >= elems) {
                double* p = c.free[i].first;
                c.free.erase(c.free.begin() + i);
                return p;
            }
    }
    double* p = nullptr;
    if (cudaHostAlloc(&p, sizeof(double) * elems, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    return p;
}
static void pin_give(double* p, size_t elems) {
    if (!p) return;
    PinCache& c = pin_cache();
    std::lock_guard<std::mutex> g(c.mu);
    if (c.free.size() < 8) c.free.emplace_back(p, elems);  // at most 8 x 32 MB kept
    else cudaFreeHost(p);
}

static int ensure_pinned(coopcg_gpu_ctx* ctx) {
    if (ctx->pin[0]) return COOPCG_OK;
    static const size_t slot_mb = [] {
        const char* e = std::getenv("COOPCG_PIN_MB");
        return e ? std::max(1, std::atoi(e)) : 32;
    }();
    const size_t slot_bytes = slot_mb << 20;
    ctx->pin_elems = std::max<size_t>(slot_bytes / sizeof(double), (size_t)ctx->n);
    for (int q = 0; q < 2; ++q) {
        ctx->pin[q] = pin_take(ctx->pin_elems);
        if (!ctx->pin[q]) return fail(ctx, COOPCG_E_CUDA, "cudaHostAlloc of the A staging slot failed");
        CK(gmalloc(ctx, &ctx->dslot[q], sizeof(double) * ctx->pin_elems, "dslot"));
        CK(cudaEventCreateWithFlags(&ctx->pin_ev[q], cudaEventDisableTiming));
    }
    return COOPCG_OK;
}

// Group handles (coopcg_gpu_create_multi) route the C ABI to their shards;
// defined at the end of this file.
static bool is_group(const coopcg_gpu_ctx* ctx) { return ctx && !ctx->shards.empty(); }
static int group_set_A(coopcg_gpu_ctx* ctx, const double* A_rows);
static int group_get_A_rows(coopcg_gpu_ctx* ctx, int row0, int rows, double* A_rows);
static int group_gen_A(coopcg_gpu_ctx* ctx, int kind, uint64_t seed, int m, double kappa);
static int group_upload(coopcg_gpu_ctx* ctx, const double* b, const double* X0);
static int group_matvec_block(coopcg_gpu_ctx* ctx, const double* D, double* out);
static int rank_gen_householder(coopcg_gpu_ctx* ctx, uint64_t seed, int m, double kappa);

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char* coopcg_gpu_version(void) { return "coopcg_gpu 2 sm_100a exact+fast"; }

int coopcg_gpu_last_error(const coopcg_gpu_ctx* ctx, char* buf, size_t len) {
    if (!buf || len == 0) return COOPCG_E_INVALID;
    const char* m = ctx ? ctx->msg.c_str() : g_create_error.c_str();
    std::snprintf(buf, len, "%s", m);
    return COOPCG_OK;
}

int coopcg_gpu_create_shard(int n, int p, int device, int arith, int row_begin, int row_end,
                            coopcg_gpu_ctx** out) {
    if (!out) return COOPCG_E_INVALID;
    *out = nullptr;
    g_create_error.clear();
    if (n < 2 || p < 1 || p >= n)
        return fail(nullptr, COOPCG_E_DIMENSION, "solver: need 1 <= p < n starting columns");  // solvers.hpp:300-306
    if (p > COOPCG_GPU_MAX_P) return fail(nullptr, COOPCG_E_DIMENSION, "p > %d agents", COOPCG_GPU_MAX_P);
    if (row_begin < 0 || row_end > n || row_begin >= row_end)
        return fail(nullptr, COOPCG_E_DIMENSION, "bad row block [%d, %d) of %d", row_begin, row_end, n);
    if (arith != COOPCG_ARITH_EXACT && arith != COOPCG_ARITH_FAST)
        return fail(nullptr, COOPCG_E_INVALID, "unknown arith mode %d", arith);
    auto* ctx = new coopcg_gpu_ctx();
    ctx->n = n;
    ctx->p = p;
    ctx->p_orig = p;
    ctx->P = (arith == COOPCG_ARITH_FAST) ? std::max(8, pad_cols(p)) : pad_cols(p);
    ctx->device = device;
    ctx->arith = arith;
    ctx->row0 = row_begin;
    ctx->row1 = row_end;
    ctx->n_loc = row_end - row_begin;
    {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
            ctx->sms = sms;
    }
    ctx->ad = pick_ad_config(ctx->n_loc, ctx->P, ctx->sms);
    if (arith == COOPCG_ARITH_FAST) {
        const int ntiles = (n + kFastT - 1) / kFastT;
        ctx->npanels = (ctx->n_loc + kFastBR - 1) / kFastBR;
        ctx->lay = ALay{1, 6, ntiles};
        ctx->ap_elems = (size_t)ctx->npanels * ntiles * kFastBR * kFastT;
        // Work units = (panel, k-chunk) on persistent CTAs (2 per SM).  Pick the
        // k-split with the best wave efficiency units/slots / ceil(units/slots)
        // (one wave for small n; e.g. n=65536: 1024 panels x 2 = 6.92 waves).
        const int slots = std::min(2 * ctx->sms, kMaxParts);
        int best_k = 1;
        double best_eff = -1.0;
        // The split is capped at 8: every extra k-chunk is one more n x P
        // partial block the row pass must sum (tools/fast_sweep.sh, round 2:
        // cap 8 vs 16: cfg 2 2861 vs 2842 it/s, cfg 1 20914 vs 19775 it/s;
        // caps 1-4 lose A.D wave efficiency).  COOPCG_FAST_KMAX overrides.
        static const int kmax = [] {
            const char* e = std::getenv("COOPCG_FAST_KMAX");
            return e ? std::max(1, std::atoi(e)) : 8;
        }();
        for (int kc = 1; kc <= std::min(kmax, ntiles); ++kc) {
            const double w = (double)ctx->npanels * kc / slots;
            const double eff = w / std::ceil(w);
            if (eff > best_eff + 1e-3) {
                best_eff = eff;
                best_k = kc;
            }
        }
        const int tpc = (ntiles + best_k - 1) / best_k;
        const int kch = (ntiles + tpc - 1) / tpc;
        ctx->f_kchunks = kch;
        ctx->f_tpc = tpc;
        ctx->f_units = ctx->npanels * kch;
        ctx->f_grid = std::min(ctx->f_units, slots);
        // Row / update passes are light; fewer CTAs keep the single-CTA
        // partial reductions short (~P^2 x grid doubles).
        const int TR = (256 / ctx->P) * 2;  // (smaller) rows per tile of fast_rows / fast_update
        static const int rg_env = [] {
            const char* e = std::getenv("COOPCG_FAST_RG");
            return e ? std::atoi(e) : 0;
        }();
        const int rg = rg_env > 0 ? std::min(rg_env, kMaxParts)
                                  : ((ctx->P <= 8) ? 128 : (ctx->P == 16 ? 192 : 296));
        // The row-pass grid fixes how the Gram partials are grouped, i.e. the rounding
        // of every p x p Gram.  On a row shard the Grams are summed over the full
        // replicated blocks and every shard must get the SAME bits (alpha, beta and
        // with them the replicated X, R, D must not drift apart between shards -- a
        // drift of one ulp grows ~100x per iteration once it starts: fast-mode solves
        // on unequal shards diverged after ~20 iterations, tools/fuzz_parity.py), so
        // the grid depends on n, not on the shard's own row count.
        ctx->f_rgrid = std::min(rg, (n + TR - 1) / TR);
        ctx->f_ugrid = std::min(rg, (n + TR - 1) / TR);
        if (ctx->n_loc == n) {
            // single GPU (the fused iteration kernel): the smallest rows-per-thread
            // whose tiles fit two co-resident CTAs per SM, one tile per CTA when
            // they do (COOPCG_FAST_RP forces 1 / 2 / 4)
            static const int rp_env = [] {
                const char* e = std::getenv("COOPCG_FAST_RP");
                return e ? std::atoi(e) : 0;
            }();
            const int slots = std::min(2 * ctx->sms, kMaxParts);
            int rp = 4;
            for (int c : {1, 2, 4})
                if ((n + (256 / ctx->P) * c - 1) / ((256 / ctx->P) * c) <= slots) {
                    rp = c;
                    break;
                }
            // no tiling gives one tile per CTA: P = 32 takes the smallest tiles (the
            // only shape whose shared memory fits two CTAs per SM), P <= 16 the largest
            if ((n + (256 / ctx->P) * rp - 1) / ((256 / ctx->P) * rp) > slots && ctx->P >= 32) rp = 1;
            if (rp_env == 1 || rp_env == 2 || rp_env == 4) rp = rp_env;
            ctx->f_rp = rp;
            const int tiles = (n + (256 / ctx->P) * rp - 1) / ((256 / ctx->P) * rp);
            ctx->f_rgrid = ctx->f_ugrid = std::min(tiles, slots);
        }
    } else {
        ctx->brs = (ctx->ad.BR == 32) ? 5 : (ctx->ad.BR == 64 ? 6 : 7);
        ctx->npanels = (ctx->n_loc + ctx->ad.BR - 1) / ctx->ad.BR;
        ctx->lay = ALay{0, ctx->brs, 0};
        ctx->ap_elems = (size_t)ctx->npanels * n * ctx->ad.BR;
    }
    set_l2_residency(ctx, 1);
    auto bail = [&](int code) {
        g_create_error = ctx->msg;
        destroy_impl(ctx);
        return code;
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        fail(ctx, COOPCG_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
        return bail(COOPCG_E_CUDA);
    }
    const size_t blk = (size_t)n * ctx->P;
#define CKC(call)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            fail(ctx, COOPCG_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
            return bail(COOPCG_E_CUDA);                                                   \
        }                                                                                 \
    } while (0)
    CKC(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CKC(gmalloc(ctx, &ctx->At, sizeof(double) * ctx->ap_elems, "A"));
    CKC(cudaMemsetAsync(ctx->At, 0, sizeof(double) * ctx->ap_elems, ctx->stream));
    double** blocks[] = {&ctx->X, &ctx->X0, &ctx->R, &ctx->Dblk[0], &ctx->Dblk[1], &ctx->Q, &ctx->S, &ctx->V};
    for (double** bp : blocks) {
        CKC(gmalloc(ctx, bp, sizeof(double) * blk, "n x P block"));
        CKC(cudaMemsetAsync(*bp, 0, sizeof(double) * blk, ctx->stream));
    }
    CKC(gmalloc(ctx, &ctx->b, sizeof(double) * n, "b"));
    if (arith == COOPCG_ARITH_FAST) {
        CKC(gmalloc(ctx, &ctx->qpart, sizeof(double) * (size_t)ctx->f_kchunks * ctx->n_loc * ctx->P, "qpart"));
        CKC(gmalloc(ctx, &ctx->gpart, sizeof(double) * (size_t)ctx->f_rgrid * 4 * ctx->P * ctx->P, "gpart"));
        CKC(gmalloc(ctx, &ctx->npart, sizeof(double) * (size_t)ctx->f_ugrid * ctx->P, "npart"));
        CKC(gmalloc(ctx, &ctx->dtiles, sizeof(double) * (size_t)ctx->lay.ntiles * ctx->P * kFastT, "dtiles"));
        CKC(gmalloc(ctx, &ctx->gfin, sizeof(double) * 4 * ctx->P * ctx->P, "gfin"));
        CKC(gmalloc(ctx, &ctx->gbar, sizeof(unsigned long long), "gbar"));
        CKC(cudaMemsetAsync(ctx->gbar, 0, sizeof(unsigned long long), ctx->stream));
        ctx->fuse_ok = ctx->n_loc == n && fast_iter_fits(ctx);
    }
    const SmallLayout L{ctx->P};
    CKC(gmalloc(ctx, &ctx->small, sizeof(double) * L.total(), "small"));
    CKC(cudaMemsetAsync(ctx->small, 0, sizeof(double) * L.total(), ctx->stream));
    ctx->nparts = kMaxParts;
    CKC(gmalloc(ctx, &ctx->partials, sizeof(double) * kMaxParts * 528, "partials"));
    CKC(gmalloc(ctx, &ctx->init_norms, sizeof(double) * (ctx->P + 1), "init_norms"));
    CKC(gmalloc(ctx, &ctx->final_norms, sizeof(double) * (ctx->P + 1), "final_norms"));
    CKC(gmalloc(ctx, &ctx->ctl, sizeof(Ctl), "ctl"));
    CKC(cudaHostAlloc(&ctx->ctl_host, 2 * sizeof(Ctl), cudaHostAllocDefault));
    CKC(cudaHostAlloc(&ctx->minres_host, 2 * kChunkMax * sizeof(double), cudaHostAllocDefault));
    std::vector<ChainDesc> descs;
    build_descs(p, ctx->P, descs, ctx->desc_off, ctx->desc_cnt);
    CKC(gmalloc(ctx, &ctx->descs, sizeof(ChainDesc) * descs.size(), "descs"));
    CKC(cudaMemcpyAsync(ctx->descs, descs.data(), sizeof(ChainDesc) * descs.size(), cudaMemcpyHostToDevice,
                        ctx->stream));
    ctx->stage_elems = std::max<size_t>(blk, (size_t)n * 128);
    CKC(gmalloc(ctx, &ctx->stage, sizeof(double) * ctx->stage_elems, "stage"));
    ctx->mv_ev.resize(2 * 2 * kChunkMax);
    for (auto& ev : ctx->mv_ev) CKC(cudaEventCreate(&ev));
    CKC(cudaEventCreate(&ctx->ev_run0));
    CKC(cudaEventCreate(&ctx->ev_run1));
    CKC(cudaEventCreate(&ctx->ev_loop0));
    CKC(cudaEventCreate(&ctx->ev_loop1));
    CKC(cudaEventCreateWithFlags(&ctx->ev_chunk[0], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_chunk[1], cudaEventDisableTiming));
    CKC(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CKC(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    // dynamic shared-memory opt-ins
    CKC(cudaFuncSetAttribute(rank_end_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)rank_smem(32)));
    CKC(cudaStreamSynchronize(ctx->stream));
#undef CKC
    *out = ctx;
    return COOPCG_OK;
}

int coopcg_gpu_create(int n, int p, int device, int arith, coopcg_gpu_ctx** out) {
    return coopcg_gpu_create_shard(n, p, device, arith, 0, n, out);
}

int coopcg_gpu_destroy(coopcg_gpu_ctx* ctx) { return destroy_impl(ctx); }

int coopcg_gpu_set_A(coopcg_gpu_ctx* ctx, const double* A_rows) {
    if (is_group(ctx)) return A_rows ? group_set_A(ctx, A_rows) : COOPCG_E_INVALID;
    if (!ctx || !A_rows) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n;
    if (int rc = ensure_pinned(ctx)) return rc;
    // Row chunks through two pinned slots: host threads fill slot s while the
    // device copies and re-lays out the chunk in slot s ^ 1.
    const int chunk = (int)std::max<size_t>(1, ctx->pin_elems / n);
    for (int c = 0, r0 = 0; r0 < ctx->n_loc; ++c, r0 += chunk) {
        const int s = c & 1;
        const int rows = std::min(chunk, ctx->n_loc - r0);
        if (c >= 2) CK(cudaEventSynchronize(ctx->pin_ev[s]));
        par_memcpy(ctx->pin[s], A_rows + (size_t)r0 * n, sizeof(double) * (size_t)rows * n);
        CK(cudaMemcpyAsync(ctx->dslot[s], ctx->pin[s], sizeof(double) * (size_t)rows * n, cudaMemcpyHostToDevice,
                           ctx->stream));
        dim3 grid((n + 31) / 32, (rows + 31) / 32);
        transpose_rows_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->dslot[s], rows, n, ctx->At, ctx->lay, r0);
        CKL();
        CK(cudaEventRecord(ctx->pin_ev[s], ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->a_ready = true;
    return COOPCG_OK;
}

int coopcg_gpu_get_A_rows(coopcg_gpu_ctx* ctx, int row0, int rows, double* A_rows) {
    if (is_group(ctx)) return A_rows ? group_get_A_rows(ctx, row0, rows, A_rows) : COOPCG_E_INVALID;
    if (!ctx || !A_rows) return COOPCG_E_INVALID;
    if (!ctx->a_ready) return fail(ctx, COOPCG_E_STATE, "A not set");
    if (row0 < 0 || rows < 0 || row0 + rows > ctx->n_loc)
        return fail(ctx, COOPCG_E_DIMENSION, "get_A_rows: row range outside this context's rows");
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n;
    if (int rc = ensure_pinned(ctx)) return rc;
    // chunk c is re-laid out and copied into pinned slot c & 1 while the host
    // threads drain chunk c - 1 from the other slot
    const int chunk = (int)std::max<size_t>(1, ctx->pin_elems / n);
    const int nch = (rows + chunk - 1) / chunk;
    for (int c = 0; c <= nch; ++c) {
        if (c < nch) {
            const int s = c & 1, r = c * chunk, m = std::min(chunk, rows - r);
            dim3 grid((n + 31) / 32, (m + 31) / 32);
            untranspose_rows_kernel<<<grid, dim3(32, 8), 0, ctx->stream>>>(ctx->At, ctx->lay, row0 + r, m, n,
                                                                          ctx->dslot[s]);
            CKL();
            CK(cudaMemcpyAsync(ctx->pin[s], ctx->dslot[s], sizeof(double) * (size_t)m * n, cudaMemcpyDeviceToHost,
                               ctx->stream));
            CK(cudaEventRecord(ctx->pin_ev[s], ctx->stream));
        }
        if (c >= 1) {
            const int s = (c - 1) & 1, r = (c - 1) * chunk, m = std::min(chunk, rows - r);
            CK(cudaEventSynchronize(ctx->pin_ev[s]));
            par_memcpy(A_rows + (size_t)r * n, ctx->pin[s], sizeof(double) * (size_t)m * n);
        }
    }
    return COOPCG_OK;
}

int coopcg_gpu_get_A(coopcg_gpu_ctx* ctx, double* A_rows) {
    if (!ctx || !A_rows) return COOPCG_E_INVALID;
    return coopcg_gpu_get_A_rows(ctx, 0, ctx->n_loc, A_rows);
}

int coopcg_gen_householder_factors(int n, int m, double kappa, uint64_t seed, double* V, double* lambda) {
    if (n < 2 || m < 0 || (!V && m > 0) || !lambda) return COOPCG_E_INVALID;
    for (int i = 0; i < n; ++i) lambda[i] = std::pow(kappa, (double)i / (double)(n - 1));
    for (int r = 0; r < m; ++r) {
        const uint64_t key = stream_key(seed, 102, (uint64_t)r);
        for (int i = 0; i < n; ++i) V[(size_t)r * n + i] = host_normal(key, (uint64_t)i);
    }
    return COOPCG_OK;
}

int coopcg_gen_rhs(int n, int kind, uint64_t seed, double* b) {
    if (n < 1 || !b) return COOPCG_E_INVALID;
    const uint64_t key = stream_key(seed, 3, (uint64_t)n);
    for (int i = 0; i < n; ++i)
        b[i] = (kind == COOPCG_VEC_UNIFORM) ? host_uniform_pm1(key, (uint64_t)i + 1) : host_normal(key, (uint64_t)i);
    return COOPCG_OK;
}

int coopcg_gen_starts(int n, int p, uint64_t seed, double* X0) {
    if (n < 1 || p < 1 || !X0) return COOPCG_E_INVALID;
    const uint64_t key = stream_key(seed, 4, (uint64_t)n);
    for (int i = 0; i < n; ++i) X0[i] = 0.0;
    for (int j = 1; j < p; ++j)
        for (int i = 0; i < n; ++i)
            X0[(size_t)j * n + i] = host_uniform_pm1(key, (uint64_t)j * (uint64_t)n + (uint64_t)i + 1);
    return COOPCG_OK;
}

int coopcg_gpu_gen_householder_begin(coopcg_gpu_ctx* ctx, uint64_t seed, int m, double kappa) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx || m < 0) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n;
    hh_free(ctx);
    std::vector<double> V((size_t)std::max(m, 1) * n), lam(n);
    coopcg_gen_householder_factors(n, m, kappa, seed, V.data(), lam.data());
    CK(gmalloc(ctx, &ctx->hh_V, sizeof(double) * V.size(), "hh_V"));
    CK(gmalloc(ctx, &ctx->hh_lam, sizeof(double) * n, "hh_lam"));
    CK(gmalloc(ctx, &ctx->hh_w, sizeof(double) * n, "hh_w"));
    CK(gmalloc(ctx, &ctx->hh_t, sizeof(double) * 2, "hh_t"));
    CK(cudaMemcpyAsync(ctx->hh_V, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->hh_lam, lam.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->hh_w, 0, sizeof(double) * n, ctx->stream));
    hh_init_kernel<<<ctx->sms * 8, 256, 0, ctx->stream>>>(ctx->At, ctx->lay, n, ctx->n_loc, ctx->row0, ctx->hh_lam,
                                                     ctx->ap_elems);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));  // the host factors are freed on return
    ctx->hh_m = m;
    ctx->a_ready = false;
    return COOPCG_OK;
}

int coopcg_gpu_gen_householder_local(coopcg_gpu_ctx* ctx, int r) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    if (ctx->hh_m < 0 || r < 0 || r >= ctx->hh_m)
        return fail(ctx, COOPCG_E_STATE, "gen_householder_local: reflector %d outside a begun generation", r);
    CK(cudaSetDevice(ctx->device));
    hh_w_kernel<<<(ctx->n_loc + 127) / 128, 128, 0, ctx->stream>>>(ctx->At, ctx->lay, ctx->n, ctx->n_loc, ctx->row0,
                                                                  ctx->hh_V + (size_t)r * ctx->n, ctx->hh_w);
    CKL();
    return COOPCG_OK;
}

int coopcg_gpu_gen_householder_rest(coopcg_gpu_ctx* ctx, int r) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    if (ctx->hh_m < 0 || r < 0 || r >= ctx->hh_m)
        return fail(ctx, COOPCG_E_STATE, "gen_householder_rest: reflector %d outside a begun generation", r);
    CK(cudaSetDevice(ctx->device));
    const double* v = ctx->hh_V + (size_t)r * ctx->n;
    hh_scalars_kernel<<<1, 32, 0, ctx->stream>>>(ctx->n, v, ctx->hh_w, ctx->hh_t);
    hh_update_kernel<<<ctx->sms * 8, 256, 0, ctx->stream>>>(ctx->At, ctx->lay, ctx->n, ctx->n_loc, ctx->row0, v, ctx->hh_w,
                                                       ctx->hh_t, ctx->ap_elems);
    CKL();
    return COOPCG_OK;
}

int coopcg_gpu_gen_householder_end(coopcg_gpu_ctx* ctx) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    if (ctx->hh_m < 0) return fail(ctx, COOPCG_E_STATE, "gen_householder_end without begin");
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    hh_free(ctx);
    ctx->a_ready = true;
    return COOPCG_OK;
}

int coopcg_gpu_gen_A(coopcg_gpu_ctx* ctx, int kind, uint64_t seed, int m, double kappa) {
    if (is_group(ctx)) return group_gen_A(ctx, kind, seed, m, kappa);
    if (!ctx) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n;
    if (kind == COOPCG_MATRIX_DIAGDOM) {
        const uint64_t key = stream_key(seed, 101, (uint64_t)n);
        gen_dd_offdiag_kernel<<<ctx->sms * 8, 256, 0, ctx->stream>>>(ctx->At, ctx->lay, n, ctx->n_loc, ctx->row0, key,
                                                                 ctx->ap_elems);
        CKL();
        gen_dd_diag_kernel<<<(ctx->n_loc + 127) / 128, 128, 0, ctx->stream>>>(ctx->At, ctx->lay, n, ctx->n_loc,
                                                                             ctx->row0);
        CKL();
    } else if (kind == COOPCG_MATRIX_HOUSEHOLDER) {
        if (ctx->n_loc != n && ctx->nccl) return rank_gen_householder(ctx, seed, m, kappa);
        if (ctx->n_loc != n)
            return fail(ctx, COOPCG_E_INVALID,
                        "row-sharded Householder generation exchanges w: use coopcg_gpu_gen_householder_*");
        if (int rc = coopcg_gpu_gen_householder_begin(ctx, seed, m, kappa)) return rc;
        for (int r = m - 1; r >= 0; --r) {
            if (int rc = coopcg_gpu_gen_householder_local(ctx, r)) return rc;
            if (int rc = coopcg_gpu_gen_householder_rest(ctx, r)) return rc;
        }
        if (int rc = coopcg_gpu_gen_householder_end(ctx)) return rc;
    } else if (kind == COOPCG_MATRIX_RANDOM_SPD) {
        if (ctx->n_loc != n) return fail(ctx, COOPCG_E_INVALID, "random_spd generation needs the full matrix");
        std::string msg;
        if (int rc = refgen_random_spd(ctx->At, ctx->lay, ctx->ap_elems, n, kappa, seed, ctx->stream, msg))
            return fail(ctx, rc, "%s", msg.c_str());
    } else {
        return fail(ctx, COOPCG_E_INVALID, "unknown matrix kind %d", kind);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->a_ready = true;
    return COOPCG_OK;
}

int coopcg_gpu_upload(coopcg_gpu_ctx* ctx, const double* b, const double* X0) {
    if (is_group(ctx)) return (b && X0) ? group_upload(ctx, b, X0) : COOPCG_E_INVALID;
    if (!ctx || !b || !X0) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n, p = ctx->p_orig, P = ctx->P;
    CK(cudaMemcpyAsync(ctx->b, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->stage, X0, sizeof(double) * (size_t)n * p, cudaMemcpyHostToDevice, ctx->stream));
    colmajor_to_rowmajor_kernel<<<grid_for((size_t)n * P, 256), 256, 0, ctx->stream>>>(ctx->stage, ctx->X0, n, p, P);
    CKL();
    ctx->inputs_ready = true;
    return COOPCG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The solve, split into phases so that a row-sharded (multi-GPU) caller can
// exchange rows between them.  "local" phases touch only this
// context's rows [row0, row1) of the output block; everything else works on
// the full, replicated n x P blocks.  A single-GPU solve runs the phases back
// to back (run_impl); sharded.py runs them with an all-gather in between.
#define LAUNCHED()              \
    do {                        \
        CKL();                  \
        ++ctx->launches;        \
    } while (0)

static bool sharded(const coopcg_gpu_ctx* ctx) { return ctx->n_loc != ctx->n; }

// Active agent count + chain descriptors for it (mccg shrinks p mid-solve).
static int set_active_p(coopcg_gpu_ctx* ctx, int p) {
    ctx->p = p;
    std::vector<ChainDesc> descs;
    build_descs(p, ctx->P, descs, ctx->desc_off, ctx->desc_cnt);
    CK(cudaMemcpyAsync(ctx->descs, descs.data(), sizeof(ChainDesc) * descs.size(), cudaMemcpyHostToDevice,
                       ctx->stream));
    return COOPCG_OK;
}

// BlockCgWorkspace::restrict_to (block_cg.hpp:84-96): keep the listed slots
// (ascending) of X, R and the given direction block; update ids / p on host
// and device.  The stream is synchronised by the caller.
static int restrict_to(coopcg_gpu_ctx* ctx, const std::vector<int>& keep, double* dir) {
    KeepList kl{};
    for (size_t c = 0; c < keep.size(); ++c) kl.keep[c] = keep[c];
    const int pk = (int)keep.size();
    const int n = ctx->n;
    double* blks[3] = {ctx->X, ctx->R, dir};
    for (double* b : blks) {
        compact_columns_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(b, n, ctx->P, kl, pk);
        CKL();
    }
    // The per-agent vectors of the small state (|D_j|^2 from the last rank
    // check, |R_j|^2, norms) are still in the old slot order: compact them
    // too, so the fast mode's SPD guard pairs each new slot's Gram diagonal
    // with its own direction norm on the first iteration after a restriction.
    {
        const SmallLayout L{ctx->P};
        const int P = ctx->P;
        std::vector<double> vec(4 * (size_t)P);
        CK(cudaMemcpyAsync(vec.data(), ctx->small + L.nsq_d(), sizeof(double) * 4 * P, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        std::vector<double> out(vec);
        for (int v = 0; v < 4; ++v)
            for (int c = 0; c < pk; ++c) out[(size_t)v * P + c] = vec[(size_t)v * P + keep[c]];
        CK(cudaMemcpyAsync(ctx->small + L.nsq_d(), out.data(), sizeof(double) * 4 * P, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    std::vector<int> nid(pk);
    for (int c = 0; c < pk; ++c) nid[c] = ctx->ids[keep[c]];
    ctx->ids = nid;
    if (int rc = set_active_p(ctx, pk)) return rc;
    Ctl& h = ctx->ctl_host[0];
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    h.p = pk;
    for (int c = 0; c < pk; ++c) h.ids[c] = nid[c];
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    return COOPCG_OK;
}

// numerical_rank(block) by the exact MGS on the device; returns rank, columns.
static int exact_rank_of(coopcg_gpu_ctx* ctx, double* blk, int& rank, std::vector<int>& cols) {
    Ctl& h = ctx->ctl_host[0];
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const int saved_stop = h.stop;
    h.force_exact = 1;
    h.stop = 0;
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    rank_end_kernel<<<1, 1024, rank_smem(ctx->P), ctx->stream>>>(ctx->partials, 1, blk, ctx->V, ctx->n, ctx->ctl, 2,
                                                                 nullptr);
    CKL();
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    rank = h.rank_result;
    cols.assign(h.rank_cols, h.rank_cols + rank);
    h.force_exact = 0;
    h.stop = saved_stop;
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    return COOPCG_OK;
}

// mccg setup_coordinator (solvers.hpp:63-98), after the device set
// restrict_pending with rank0 (and its columns when rank0 < p).
static int mccg_setup(coopcg_gpu_ctx* ctx) {
    Ctl& h = ctx->ctl_host[0];
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const int p = ctx->p;
    const int rank0 = h.rank_result;
    std::vector<double> init(p + 1);
    CK(cudaMemcpy(init.data(), ctx->init_norms, sizeof(double) * (p + 1), cudaMemcpyDeviceToHost));
    std::vector<int> keep(p);
    for (int j = 0; j < p; ++j) keep[j] = j;
    if (rank0 > 0 && rank0 < p) {
        keep.assign(h.rank_cols, h.rank_cols + rank0);
        std::sort(keep.begin(), keep.end());
        if (int rc = restrict_to(ctx, keep, ctx->Dblk[0])) return rc;
    }
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    h.restrict_pending = 0;
    int slot = -1;
    for (int j = 0; j < (int)keep.size(); ++j)
        if (init[keep[j]] <= h.tol) {
            slot = j;
            break;
        }
    if (slot >= 0) {
        h.status = COOPCG_CONVERGED;
        h.converged_agent = ctx->ids[slot];
        h.stop = 1;
    } else if (rank0 == 0) {
        ctx->host_err = COOPCG_E_NUMERICAL_BREAKDOWN;
        ctx->host_err_msg = "every starting direction is numerically zero";  // solvers.hpp:86-91
        h.stop = 1;
    }
    if (!h.stop && h.max_iters == 0) {
        h.status = COOPCG_MAX_ITERATIONS;
        h.stop = 1;
    }
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return COOPCG_OK;
}

// mccg end_of_iteration restriction (solvers.hpp:156-185) for iteration kr,
// whose D' block is Dblk[(kr+1)&1].  Returns the next k (or -1 when stopped).
static int mccg_restrict(coopcg_gpu_ctx* ctx, int kr, int* next_k) {
    Ctl& h = ctx->ctl_host[0];
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const int rr = h.rank_result;
    int nsel = 0;
    std::vector<int> cols;
    if (int rc = exact_rank_of(ctx, ctx->R, nsel, cols)) return rc;
    const int pnext = std::min(rr, nsel);
    *next_k = -1;
    if (pnext == 0) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "all agents degenerate at iteration %d with residual above tolerance", kr);
        ctx->host_err = COOPCG_E_NUMERICAL_BREAKDOWN;
        ctx->host_err_msg = buf;
        CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        h.restrict_pending = 0;
        h.stop = 1;
        CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
        return COOPCG_OK;
    }
    std::vector<int> keep(cols.begin(), cols.begin() + pnext);
    std::sort(keep.begin(), keep.end());
    if (int rc = restrict_to(ctx, keep, ctx->Dblk[(kr + 1) & 1])) return rc;
    CK(cudaMemcpyAsync(&h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    h.restrict_pending = 0;
    if (kr + 1 >= h.max_iters) {
        h.status = COOPCG_MAX_ITERATIONS;
        h.stop = 1;
    } else {
        h.k = kr + 1;
        h.stop = 0;
        *next_k = kr + 1;
    }
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return COOPCG_OK;
}
static int dgrid_of(const coopcg_gpu_ctx* ctx) {
    if (ctx->arith == COOPCG_ARITH_FAST) return ctx->f_ugrid;
    return exact_dgrid(ctx);
}

// fast_rows over arbitrary (Qpart, kchunks, rows) -- the local row pass or a
// full-n Gram pass over a replicated block (Qpart = the block itself).
template <int P>
cudaError_t fast_rows_any_t(coopcg_gpu_ctx* ctx, const double* qpart, int kchunks, int nrows, int row0, double* dst,
                            const double* b, const double* D, const double* R, const double* Qfull, int mode,
                            const int* stop) {
    pdl_launch(fast_rows_kernel<P>, dim3(ctx->f_rgrid), dim3(256), 0, ctx->stream, qpart, kchunks, nrows, row0, dst, b, D, R, Qfull,
               ctx->p, mode, ctx->gpart, stop, PeerRows{});
    ++ctx->launches;
    return cudaGetLastError();
}
static cudaError_t fast_rows_any(coopcg_gpu_ctx* ctx, const double* qpart, int kchunks, int nrows, int row0,
                                 double* dst, const double* b, const double* D, const double* R,
                                 const double* Qfull, int mode, const int* stop) {
    switch (ctx->P) {
    case 8: return fast_rows_any_t<8>(ctx, qpart, kchunks, nrows, row0, dst, b, D, R, Qfull, mode, stop);
    case 16: return fast_rows_any_t<16>(ctx, qpart, kchunks, nrows, row0, dst, b, D, R, Qfull, mode, stop);
    default: return fast_rows_any_t<32>(ctx, qpart, kchunks, nrows, row0, dst, b, D, R, Qfull, mode, stop);
    }
}

// ---- verification mode (keep_history / x_star) --------------------------------
// Buffers for the coming solve; refuses what the mode does not cover.
static int ver_begin(coopcg_gpu_ctx* ctx) {
    ctx->ver_iters = -1;
    if (!ctx->ver_hist_on && !ctx->ver_xs_on) return COOPCG_OK;
    if (ctx->algo == 1)
        return fail(ctx, COOPCG_E_INVALID, "keep_history / x_star are not available with mccg_solve on the GPU");
    const size_t blk = (size_t)ctx->n * ctx->P;
    if (ctx->ver_hist_on) {
        const int entries = ctx->max_iters + 1;
        if (entries > ctx->ver_hist_cap) {
            gfree(ctx, ctx->ver_hist);
            ctx->ver_hist = nullptr;
            ctx->ver_hist_cap = 0;
            const size_t bytes = sizeof(double) * 3 * blk * (size_t)entries;
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            if (bytes > free_b / 2)
                return fail(ctx, COOPCG_E_INVALID,
                            "keep_history: %d entries of three %d x %d blocks need %.1f GB of device memory "
                            "(set max_iters)", entries, ctx->n, ctx->p, bytes / 1e9);
            CK(gmalloc(ctx, &ctx->ver_hist, bytes, "ver_hist"));
            ctx->ver_hist_cap = entries;
        }
    }
    if (ctx->ver_xs_on) {
        if (!ctx->ver_E) CK(gmalloc(ctx, &ctx->ver_E, sizeof(double) * blk, "ver_E"));
        if (!ctx->ver_AE) CK(gmalloc(ctx, &ctx->ver_AE, sizeof(double) * blk, "ver_AE"));
        if (!ctx->ver_flag) CK(gmalloc(ctx, &ctx->ver_flag, sizeof(int), "ver_flag"));
        const int rows = std::max(ctx->max_iters, 1);
        if (rows > ctx->ver_anorm_cap) {
            gfree(ctx, ctx->ver_anorm);
            ctx->ver_anorm = nullptr;
            ctx->ver_anorm_cap = 0;
            CK(gmalloc(ctx, &ctx->ver_anorm, sizeof(double) * (size_t)rows * ctx->p_orig, "ver_anorm"));
            ctx->ver_anorm_cap = rows;
        }
        CK(cudaMemsetAsync(ctx->ver_flag, 0, sizeof(int), ctx->stream));
    }
    return COOPCG_OK;
}
// History entry `entry` <- (X, R, dir): push_history (solvers.hpp:43-50).  Entries
// enqueued after a device-side stop copy unchanged blocks and are never read.
static int ver_snapshot(coopcg_gpu_ctx* ctx, int entry, const double* dir) {
    if (!ctx->ver_hist_on || entry >= ctx->ver_hist_cap) return COOPCG_OK;
    const size_t blk = (size_t)ctx->n * ctx->P;
    double* h = ctx->ver_hist + (size_t)entry * 3 * blk;
    CK(cudaMemcpyAsync(h, ctx->X, sizeof(double) * blk, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(h + blk, ctx->R, sizeof(double) * blk, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(h + 2 * blk, dir, sizeof(double) * blk, cudaMemcpyDeviceToDevice, ctx->stream));
    return COOPCG_OK;
}
// Row k of the A-norm errors: ||x_j - x*||_A per agent after iteration k's update
// (anorm_errors, block_cg.hpp:316-331).  No stop check: the iteration that raises
// the stop still records (solvers.hpp:131); later launches write unread rows.
static int ver_anorm(coopcg_gpu_ctx* ctx, int k) {
    if (!ctx->ver_xs_on || k >= ctx->ver_anorm_cap) return COOPCG_OK;
    const int n = ctx->n, P = ctx->P;
    cudaStream_t st = ctx->stream;
    ver_diff_kernel<<<grid_for((size_t)n * P, 256), 256, 0, st>>>(ctx->X, ctx->ver_xs, ctx->ver_E, n, ctx->p, P);
    LAUNCHED();
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(ad_launch(ctx, ctx->ver_E, ctx->ver_AE, nullptr, nullptr));
    } else {
        CK(fast_ad(ctx, ctx->ver_E, nullptr));
        CK(fast_rows(ctx, ctx->ver_AE, nullptr, nullptr, nullptr, nullptr, 1, nullptr));
    }
    ver_anorm_kernel<<<1, 256, sizeof(double) * 2 * kVerTile * P, st>>>(
        ctx->ver_E, ctx->ver_AE, n, ctx->p, P, ctx->ver_anorm + (size_t)k * ctx->p_orig, ctx->ver_flag);
    LAUNCHED();
    return COOPCG_OK;
}

static int begin_impl(coopcg_gpu_ctx* ctx, const coopcg_opts* opts) {
    if (!ctx->a_ready) return fail(ctx, COOPCG_E_STATE, "A not set (coopcg_gpu_set_A / coopcg_gpu_gen_A)");
    if (!ctx->inputs_ready) return fail(ctx, COOPCG_E_STATE, "b / X0 not uploaded");
    coopcg_opts o{0.0, -1, -1, 1e-10};
    if (opts) o = *opts;
    ctx->max_iters = o.max_iters >= 0 ? o.max_iters : 2 * ctx->n;  // solvers.hpp:18-23
    ctx->every = o.recompute_residual_every >= 0 ? o.recompute_residual_every : 50;
    if (int rc = ensure_trace_capacity(ctx, std::max(ctx->max_iters, 1))) return rc;
    ctx->algo = (o.algo == 1 || o.algo == 2) ? o.algo : 0;
    if (ctx->algo == 2 && (ctx->p != 1 || ctx->arith != COOPCG_ARITH_EXACT))
        return fail(ctx, COOPCG_E_INVALID, "steepest descent needs p = 1 and the exact mode");
    if (int rc = ver_begin(ctx)) return rc;
    ctx->host_err = 0;
    ctx->host_err_msg.clear();
    if (ctx->p != ctx->p_orig)
        if (int rc = set_active_p(ctx, ctx->p_orig)) return rc;
    ctx->ids.resize(ctx->p_orig);
    for (int j = 0; j < ctx->p_orig; ++j) ctx->ids[j] = j;
    Ctl h{};
    h.stop = 0;
    h.status = COOPCG_MAX_ITERATIONS;
    h.k = 0;
    h.converged_agent = -1;
    h.tol = o.tol;
    h.rank_rel_tol = o.rank_rel_tol;
    h.max_iters = ctx->max_iters;
    h.p = ctx->p;
    h.P = ctx->P;
    h.algo = ctx->algo;
    h.p0 = ctx->p_orig;
    for (int j = 0; j < ctx->p_orig; ++j) h.ids[j] = j;
    std::memcpy(&ctx->ctl_host[0], &h, sizeof(Ctl));
    CK(cudaMemcpyAsync(ctx->ctl, &ctx->ctl_host[0], sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream));
    // every solve starts from the uploaded X0 (the previous solve overwrote X)
    CK(cudaMemcpyAsync(ctx->X, ctx->X0, sizeof(double) * (size_t)ctx->n * ctx->P, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    ctx->launches = 0;
    ctx->phase_mv = 0;
    return COOPCG_OK;
}

// R_loc = A_loc X - b (stage_setup, block_cg.hpp:132-138)
static int setup_local(coopcg_gpu_ctx* ctx) {
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(ad_launch(ctx, ctx->X, ctx->R, ctx->b, nullptr));
    } else {
        CK(fast_ad(ctx, ctx->X, nullptr));
        CK(fast_rows(ctx, ctx->R, ctx->b, nullptr, nullptr, nullptr, 1, nullptr));
    }
    return COOPCG_OK;
}

// D = R, norms, tolerance and rank checks (block_cg.hpp:139-144, solvers.hpp:55-100)
static int setup_rest(coopcg_gpu_ctx* ctx) {
    const int n = ctx->n, P = ctx->P;
    cudaStream_t st = ctx->stream;
    int* stop = &ctx->ctl->stop;
    const bool fast = ctx->arith == COOPCG_ARITH_FAST;
    CK(cudaMemcpyAsync(ctx->Dblk[0], ctx->R, sizeof(double) * (size_t)n * P, cudaMemcpyDeviceToDevice, st));
    if (!fast) {
        CK(chains_launch(ctx, kPhSetup, ctx->R, nullptr, nullptr, 1, nullptr));
        setup_norms_kernel<<<1, 32, 0, st>>>(ctx->small, ctx->ctl, ctx->init_norms);
    } else {
        if (sharded(ctx))  // full-n residual norms over the replicated R
            CK(fast_rows_any(ctx, ctx->R, 1, n, 0, ctx->R, nullptr, nullptr, nullptr, nullptr, 1, nullptr));
        fast_norms_kernel<<<1, 256, 0, st>>>(ctx->gpart, ctx->f_rgrid, 4 * P * P, P * P, P + 1, ctx->ctl,
                                             ctx->init_norms, 1, ctx->small);
    }
    LAUNCHED();
    const int dgrid = dgrid_of(ctx);
    CK(gram_partials_launch(ctx, ctx->Dblk[0], dgrid, stop));
    ++ctx->launches;
    rank_end_kernel<<<1, 1024, rank_smem(P), st>>>(ctx->partials, dgrid, ctx->Dblk[0], ctx->V, n, ctx->ctl, 1,
                                                   fast ? ctx->small : nullptr);
    LAUNCHED();
    return COOPCG_OK;
}

// Q_loc = A_loc D_k  (stage_matvec, block_cg.hpp:146-151), bracketed by events.
// Q of iteration k: double-buffered by parity in peer mode (see Qalt).
static double* q_of(const coopcg_gpu_ctx* ctx, int k) { return (ctx->p2p && (k & 1)) ? ctx->Qalt : ctx->Q; }
static PeerRows peers_of(const coopcg_gpu_ctx* ctx, int k) { return ctx->p2p ? ctx->peers[k & 1] : PeerRows{}; }

// Make the main stream wait for an outstanding side-stream rank_end.
static int join_rank(coopcg_gpu_ctx* ctx) {
    if (!ctx->join_pending) return COOPCG_OK;
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
    ctx->join_pending = false;
    return COOPCG_OK;
}

static bool recompute_at(const coopcg_gpu_ctx* ctx, int k) {
    return ctx->every > 0 && (k + 1) % ctx->every == 0;  // solvers.hpp:33-35
}

static int iter_local(coopcg_gpu_ctx* ctx, int k, cudaEvent_t ev0, cudaEvent_t ev1) {
    double* Qk = q_of(ctx, k);
    int* stop = &ctx->ctl->stop;
    double* D = ctx->Dblk[k & 1];
    if (ev0) CK(cudaEventRecord(ev0, ctx->stream));
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(ad_launch(ctx, D, Qk, nullptr, stop, peers_of(ctx, k)));
        if (ev1) CK(cudaEventRecord(ev1, ctx->stream));
        if (int rc = join_rank(ctx)) return rc;
    } else {
        CK(fast_ad(ctx, D, stop));
        if (ev1) CK(cudaEventRecord(ev1, ctx->stream));
        if (int rc = join_rank(ctx)) return rc;
        if (!sharded(ctx) && !recompute_at(ctx, k) && ctx->fuse_ok && fuse_enabled()) {
            // single GPU, plain iteration: row pass + Grams + solves + update in one launch
            CK(fast_iter(ctx, Qk, D, ctx->Dblk[(k + 1) & 1]));
            ctx->fused_k = k;
        } else {
            ctx->fused_k = -1;
            // single GPU: fuse the four Gram partials into the local row pass
            CK(fast_rows(ctx, Qk, nullptr, D, ctx->R, nullptr, sharded(ctx) ? 1 : 0, stop, peers_of(ctx, k)));
        }
    }
    return COOPCG_OK;
}


// After Q is complete: Grams, alpha, update; in recompute iterations ends with
// R_loc = A_loc X - b (the caller exchanges R before iter_rest).
static int iter_mid(coopcg_gpu_ctx* ctx, int k) {
    double* Qk = q_of(ctx, k);
    const int n = ctx->n;
    int* stop = &ctx->ctl->stop;
    double* D = ctx->Dblk[k & 1];
    double* Dn = ctx->Dblk[(k + 1) & 1];
    const bool rec = recompute_at(ctx, k);
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(chains_launch(ctx, kPhGram, D, Qk, ctx->R, 3, stop));
        CK(alpha_update_launch(ctx, Qk, D, rec ? 1 : 0));
        if (rec) CK(ad_launch(ctx, ctx->X, ctx->R, ctx->b, stop));
    } else {
        if (sharded(ctx))  // the four Gram partials over the full replicated blocks
            CK(fast_rows_any(ctx, Qk, 1, n, 0, Qk, nullptr, D, ctx->R, nullptr, 0, stop));
        if (!rec) {
            if (ctx->fused_k != k) {
                CK(fast_solve(ctx, 0));
                CK(fast_update(ctx, Qk, D, Dn, 0, stop));  // the record follows in iter_rest
            }
        } else {
            CK(fast_solve(ctx, 1));
            CK(fast_update(ctx, Qk, D, Dn, 1, stop));
            CK(fast_ad(ctx, ctx->X, stop));
            // local rows of R = A X - b (with R^T Q / |R|^2 partials when unsharded)
            CK(fast_rows(ctx, ctx->R, ctx->b, nullptr, nullptr, sharded(ctx) ? nullptr : Qk, 1, stop));
        }
    }
    return COOPCG_OK;
}

// The rest of the iteration: beta, D', norms/record, rank check, k++.
static int iter_rest(coopcg_gpu_ctx* ctx, int k) {
    double* Qk = q_of(ctx, k);
    const int n = ctx->n, P = ctx->P;
    cudaStream_t st = ctx->stream;
    int* stop = &ctx->ctl->stop;
    double* D = ctx->Dblk[k & 1];
    double* Dn = ctx->Dblk[(k + 1) & 1];
    const bool rec = recompute_at(ctx, k);
    const bool fast = ctx->arith == COOPCG_ARITH_FAST;
    if (!fast) {
        CK(chains_launch(ctx, kPhBeta, ctx->R, Qk, nullptr, 2, stop));
        CK(beta_direction_launch(ctx, D, Dn));
    } else if (rec) {
        if (sharded(ctx))  // R^T Q and |R|^2 over the full replicated, recomputed R
            CK(fast_rows_any(ctx, ctx->R, 1, n, 0, ctx->R, nullptr, nullptr, nullptr, Qk, 1, stop));
        CK(fast_solve(ctx, 2));
        CK(fast_update(ctx, Qk, D, Dn, 2, stop));
    }
    // The record (fast mode) and the rank certificate of D' gate only what
    // comes after the next A.D (which reads D' and nothing they write): in
    // run_impl they run on the side stream, concurrently with that A.D.  A
    // stop they raise turns the rest of the iteration into no-ops as before;
    // the A.D they overlapped only wrote scratch.
    cudaStream_t rs = st;
    if (ctx->rank_async) {
        CK(cudaEventRecord(ctx->ev_fork, st));
        CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
        rs = ctx->side;
    }
    if (fast) {
        // norms -> record + convergence (solvers.hpp:125-154), then k++ in rank_end
        if (!rec)
            pdl_launch(fast_record_kernel, dim3(1), dim3(256), 0, rs, ctx->npart, ctx->f_ugrid, P, 0, 1, ctx->small,
                       ctx->ctl, ctx->tr_norms, ctx->tr_minres, ctx->tr_wall, ctx->tr_capacity);
        else
            pdl_launch(fast_record_kernel, dim3(1), dim3(256), 0, rs, ctx->gpart, ctx->f_rgrid, 4 * P * P, P * P, P + 1,
                       ctx->small, ctx->ctl, ctx->tr_norms, ctx->tr_minres, ctx->tr_wall, ctx->tr_capacity);
        LAUNCHED();
    }
    pdl_launch(rank_end_kernel, dim3(1), dim3(1024), rank_smem(P), rs, ctx->partials, dgrid_of(ctx), Dn, ctx->V, n, ctx->ctl, 0,
                                                   fast ? ctx->small : nullptr);
    LAUNCHED();
    if (ctx->rank_async) {
        CK(cudaEventRecord(ctx->ev_join, ctx->side));
        ctx->join_pending = true;
    }
    return COOPCG_OK;
}

// S_loc = A_loc X - b (finalize_trace, solvers.hpp:196-205)
static int final_local(coopcg_gpu_ctx* ctx) {
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(ad_launch(ctx, ctx->X, ctx->S, ctx->b, nullptr));
    } else {
        CK(fast_ad(ctx, ctx->X, nullptr));
        CK(fast_rows(ctx, ctx->S, ctx->b, nullptr, nullptr, nullptr, 1, nullptr));
    }
    return COOPCG_OK;
}

static int final_rest(coopcg_gpu_ctx* ctx) {
    const int n = ctx->n, P = ctx->P;
    cudaStream_t st = ctx->stream;
    if (ctx->arith != COOPCG_ARITH_FAST) {
        CK(chains_launch(ctx, kPhFinal, ctx->S, nullptr, nullptr, 1, nullptr));
        final_norms_kernel<<<1, 32, 0, st>>>(ctx->small, ctx->ctl, ctx->final_norms);
    } else {
        if (sharded(ctx))
            CK(fast_rows_any(ctx, ctx->S, 1, n, 0, ctx->S, nullptr, nullptr, nullptr, nullptr, 1, nullptr));
        fast_norms_kernel<<<1, 256, 0, st>>>(ctx->gpart, ctx->f_rgrid, 4 * P * P, P * P, P + 1, ctx->ctl,
                                             ctx->final_norms, 0, ctx->small);
    }
    LAUNCHED();
    return COOPCG_OK;
}

// Copy the trace out: one read of the control block, then every trace piece
// (and the final X) enqueued as async copies into pinned staging and a single
// synchronisation (pageable cudaMemcpy calls cost a host round trip each).
static int end_impl(coopcg_gpu_ctx* ctx, coopcg_trace* trace) {
    const int n = ctx->n, p = ctx->p, P = ctx->P;
    cudaStream_t st = ctx->stream;
    CK(cudaMemcpyAsync(&ctx->ctl_host[0], ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const Ctl& fin = ctx->ctl_host[0];
    if (trace) {
        const int iters = fin.iterations;
        const int p0 = ctx->p_orig;
        trace->status = fin.status;
        trace->converged_agent = fin.converged_agent;
        trace->iterations = iters;
        trace->exact_rank_checks = fin.exact_rank_checks;
        const int cap = std::min(iters, trace->capacity);
        // staging layout: wall[iters] | init[p0+1] | final[p+1] | norms[cap*p0] | minres[cap]
        const size_t n_wall = (size_t)std::max(iters, 0), n_init = p0 + 1, n_fin = p + 1;
        const size_t n_norm = (trace->residual_norms && cap > 0) ? (size_t)cap * p0 : 0;
        const size_t n_min = (trace->minres && cap > 0) ? (size_t)cap : 0;
        const size_t bytes = 8 * (n_wall + n_init + n_fin + n_norm + n_min);
        if (bytes > ctx->trace_host_bytes) {
            if (ctx->trace_host) cudaFreeHost(ctx->trace_host);
            ctx->trace_host = nullptr;
            ctx->trace_host_bytes = 0;
            CK(cudaHostAlloc(&ctx->trace_host, bytes, cudaHostAllocDefault));
            ctx->trace_host_bytes = bytes;
        }
        auto* wall = reinterpret_cast<unsigned long long*>(ctx->trace_host);
        double* init = reinterpret_cast<double*>(wall + n_wall);
        double* finl = init + n_init;
        double* norms = finl + n_fin;
        double* minres = norms + n_norm;
        if (n_wall) CK(cudaMemcpyAsync(wall, ctx->tr_wall, 8 * n_wall, cudaMemcpyDeviceToHost, st));
        // initial norms were recorded before any restriction (p_orig entries)
        CK(cudaMemcpyAsync(init, ctx->init_norms, 8 * n_init, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(finl, ctx->final_norms, 8 * n_fin, cudaMemcpyDeviceToHost, st));
        if (n_norm)  // rows of p_orig, NaN for inactive agents
            CK(cudaMemcpyAsync(norms, ctx->tr_norms, 8 * n_norm, cudaMemcpyDeviceToHost, st));
        if (n_min) CK(cudaMemcpyAsync(minres, ctx->tr_minres, 8 * n_min, cudaMemcpyDeviceToHost, st));
        const bool scatter = p != p0;
        std::vector<double> xs;
        if (trace->final_x) {
            rowmajor_to_colmajor_kernel<<<grid_for((size_t)n * p, 256), 256, 0, st>>>(ctx->X, ctx->stage, n, p, P);
            CKL();
            if (!scatter) {
                CK(cudaMemcpyAsync(trace->final_x, ctx->stage, sizeof(double) * (size_t)n * p, cudaMemcpyDeviceToHost,
                                   st));
            } else {
                xs.resize((size_t)n * p);
                CK(cudaMemcpyAsync(xs.data(), ctx->stage, sizeof(double) * xs.size(), cudaMemcpyDeviceToHost, st));
            }
        }
        CK(cudaStreamSynchronize(st));
        uint64_t total = 0;
        for (int k = 0; k < iters; ++k) total += wall[k];
        trace->loop_wall_ns = total;
        if (n_norm) std::memcpy(trace->residual_norms, norms, 8 * n_norm);
        if (n_min) std::memcpy(trace->minres, minres, 8 * n_min);
        if (trace->wall_ns && cap > 0) std::memcpy(trace->wall_ns, wall, sizeof(uint64_t) * cap);
        if (trace->initial_residual_norms) std::memcpy(trace->initial_residual_norms, init, sizeof(double) * p0);
        trace->initial_minres = init[p0];
        trace->final_minres = finl[p];
        if (trace->final_residual_norms) {
            if (!scatter) {
                std::memcpy(trace->final_residual_norms, finl, sizeof(double) * p);
            } else {  // mccg: per original agent id, NaN for dropped agents
                for (int j = 0; j < p0; ++j) trace->final_residual_norms[j] = std::nan("");
                for (int j = 0; j < p; ++j) trace->final_residual_norms[ctx->ids[j]] = finl[j];
            }
        }
        if (trace->active_agents)
            for (int j = 0; j < p; ++j) trace->active_agents[j] = ctx->ids[j];
        trace->n_active = p;
        if (trace->final_x && scatter) {
            for (size_t e = 0; e < (size_t)n * p0; ++e) trace->final_x[e] = std::nan("");
            for (int j = 0; j < p; ++j)
                std::memcpy(trace->final_x + (size_t)ctx->ids[j] * n, xs.data() + (size_t)j * n, sizeof(double) * n);
        }
    }
    if (ctx->ver_hist_on || ctx->ver_xs_on) {
        ctx->ver_iters = fin.iterations;
        // Exact mode forms D' only when the iteration goes on (beta_direction_kernel
        // returns once an agent has converged); the reference forms Dnext before
        // end_of_iteration and pushes it (solvers.hpp:146), so the converging
        // iteration's history entry gets its direction block here: D' = R + D beta^T
        // with the beta the iteration solved (D' = R for steepest descent).
        if (ctx->ver_hist_on && ctx->arith != COOPCG_ARITH_FAST && fin.status == 0 && fin.iterations >= 1 &&
            fin.iterations < ctx->ver_hist_cap) {
            const int ks = fin.iterations - 1;
            const size_t blk = (size_t)n * P;
            const SmallLayout L{P};
            ver_direction_kernel<<<grid_for(blk, 256), 256, 0, st>>>(
                ctx->R, ctx->Dblk[ks & 1], ctx->small + L.beta(), ctx->ver_hist + ((size_t)(ks + 1) * 3 + 2) * blk, n, p,
                P, ctx->algo == 2 ? 1 : 0);
            CKL();
            CK(cudaStreamSynchronize(st));
        }
        if (ctx->ver_xs_on && ctx->ver_flag) {
            int flag = 0;
            CK(cudaMemcpyAsync(&flag, ctx->ver_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (flag)  // dense_ops.hpp:190-191
                return fail(ctx, COOPCG_E_SPD_VIOLATION, "a_norm: quadratic form negative beyond round-off");
        }
    }
    if (ctx->host_err) return fail(ctx, ctx->host_err, "%s", ctx->host_err_msg.c_str());
    if (fin.err == COOPCG_E_SPD_VIOLATION)
        return fail(ctx, COOPCG_E_SPD_VIOLATION, "nonpositive direction energy d^T A d at iteration %d",
                    fin.err_iter);  // solvers.hpp:111-115
    return COOPCG_OK;
}

// ---------------------------------------------------------------------------
// Row exchanges between the shards of a solve.  One solve is
// run by a set of LOCAL contexts (the shards this process drives) under one of
//   mode 0  one context holding every row (nothing to exchange),
//   mode 1  shards of one process (coopcg_gpu_create_multi): Q rows are pushed
//           into every shard's Q by the kernel that computes them (peer
//           stores over NVLink, or plain stores when shards share a device)
//           and the exchange is a cross-stream event barrier; R / S / w rows
//           are peer copies between two barriers,
//   mode 2  one rank context per process (coopcg_gpu_create_rank): every row
//           exchange is an all-gather of the row blocks (grouped in-place NCCL
//           broadcasts, one per rank) on the context stream.
// Everything is stream-ordered: the host enqueues whole chunks of iterations
// for every shard and reads one control snapshot per chunk, as for one GPU.
struct Exch {
    int mode = 0;
    std::vector<coopcg_gpu_ctx*> s;        // local shards, rank order (s[0] records the trace)
    std::vector<cudaEvent_t>* ev = nullptr; // mode 1: one barrier event per shard
};

static Exch exch_of(coopcg_gpu_ctx* ctx) {
    Exch X;
    if (!ctx->shards.empty()) {
        X.mode = 1;
        X.s = ctx->shards;
        X.ev = &ctx->gev;
    } else {
        X.mode = ctx->nccl ? 2 : 0;
        X.s = {ctx};
    }
    return X;
}

// Run f on every local shard (its device current); a failure's message is
// copied to the handle h.
template <typename F>
static int each(coopcg_gpu_ctx* h, const Exch& X, F&& f) {
    for (coopcg_gpu_ctx* c : X.s) {
        if (X.s.size() > 1 || c != h) {
            cudaError_t e = cudaSetDevice(c->device);
            if (e != cudaSuccess) return fail(h, COOPCG_E_CUDA, "cudaSetDevice(%d): %s", c->device, cudaGetErrorString(e));
        }
        if (int rc = f(c)) {
            if (c != h) h->msg = c->msg;
            return rc;
        }
    }
    return COOPCG_OK;
}

// mode 1: every shard's stream waits for every other shard's current position.
static int xbarrier(coopcg_gpu_ctx* ctx, const Exch& X) {
    if (X.mode != 1 || X.s.size() < 2) return COOPCG_OK;
    for (size_t g = 0; g < X.s.size(); ++g) {
        CK(cudaSetDevice(X.s[g]->device));
        CK(cudaEventRecord((*X.ev)[g], X.s[g]->stream));
    }
    for (size_t h = 0; h < X.s.size(); ++h) {
        CK(cudaSetDevice(X.s[h]->device));
        for (size_t g = 0; g < X.s.size(); ++g)
            if (g != h) CK(cudaStreamWaitEvent(X.s[h]->stream, (*X.ev)[g], 0));
    }
    return COOPCG_OK;
}

// Device buffer of block `which` (n rows, ld doubles per row) on shard c.
static double* block_of(coopcg_gpu_ctx* c, int which, int k, int* ld) {
    *ld = c->P;
    switch (which) {
    case COOPCG_BLOCK_R: return c->R;
    case COOPCG_BLOCK_Q: return (c->p2p && (k & 1)) ? c->Qalt : c->Q;
    case COOPCG_BLOCK_S: return c->S;
    case COOPCG_BLOCK_W: *ld = 1; return c->hh_w;
    default: return nullptr;
    }
}

static const char* nccl_err(ncclResult_t r) {
    const NcclApi& api = nccl_api();
    return api.errorString ? api.errorString(r) : "nccl error";
}

// All-gather of the row blocks of `which`: afterwards every shard holds every
// shard's rows [row0, row1).
static int xrows(coopcg_gpu_ctx* ctx, const Exch& X, int which, int k) {
    if (X.mode == 0) return COOPCG_OK;
    if (X.mode == 2) {
        coopcg_gpu_ctx* c = X.s[0];
        const NcclApi& api = nccl_api();
        int ld = 0;
        double* buf = block_of(c, which, k, &ld);
        ncclResult_t r = api.groupStart();
        for (int q = 0; q < c->nranks && r == ncclSuccess; ++q) {
            int r0 = 0, r1 = 0;
            row_split(c->n, c->nranks, q, &r0, &r1);
            if (r1 > r0)
                r = api.broadcast(buf + (size_t)r0 * ld, buf + (size_t)r0 * ld, (size_t)(r1 - r0) * ld, ncclFloat64,
                                  q, static_cast<ncclComm_t>(c->nccl), c->stream);
        }
        ncclResult_t r2 = api.groupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(ctx, COOPCG_E_CUDA, "NCCL all-gather of rows: %s", nccl_err(r != ncclSuccess ? r : r2));
        return COOPCG_OK;
    }
    if (X.s.size() < 2) return COOPCG_OK;
    // every shard has reached the exchange (no later write of a peer's rows
    // can race with the copies), copies, and every copy has landed
    if (int rc = xbarrier(ctx, X)) return rc;
    for (coopcg_gpu_ctx* g : X.s) {
        CK(cudaSetDevice(g->device));
        int ld = 0;
        const double* src = block_of(g, which, k, &ld) + (size_t)g->row0 * ld;
        const size_t bytes = sizeof(double) * (size_t)g->n_loc * ld;
        for (coopcg_gpu_ctx* h : X.s)
            if (h != g)
                CK(cudaMemcpyPeerAsync(block_of(h, which, k, &ld) + (size_t)g->row0 * ld, h->device, src, g->device,
                                       bytes, g->stream));
    }
    return xbarrier(ctx, X);
}

// After every shard's iter_local(k): the full Q of iteration k everywhere.
static int xq(coopcg_gpu_ctx* ctx, const Exch& X, int k) {
    if (X.mode == 1) return xbarrier(ctx, X);  // the rows were pushed by the producing kernel
    return xrows(ctx, X, COOPCG_BLOCK_Q, k);
}

static int run_impl(coopcg_gpu_ctx* ctx, const coopcg_opts* opts, coopcg_trace* trace) {
    const Exch X = exch_of(ctx);
    coopcg_gpu_ctx* c0 = X.s[0];
    if (X.mode == 0 && sharded(c0))
        return fail(ctx, COOPCG_E_STATE,
                    "a row shard without an exchange is driven phase by phase (coopcg_gpu_phase); "
                    "use coopcg_gpu_create_multi / coopcg_gpu_create_rank for a multi-GPU run");
    if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return begin_impl(c, opts); })) return rc;
    auto on0 = [&]() -> int {
        CK(cudaSetDevice(c0->device));
        return COOPCG_OK;
    };
    const int max_iters = c0->max_iters;
    if (int rc = on0()) return rc;
    CK(cudaEventRecord(c0->ev_run0, c0->stream));
    if (int rc = each(ctx, X, setup_local)) return rc;
    if (int rc = xrows(ctx, X, COOPCG_BLOCK_R, 0)) return rc;
    if (int rc = each(ctx, X, setup_rest)) return rc;
    // verification mode (one context holding every row): history entry 0 = the
    // state after setup; everything stays on the main stream (the A-norm pass
    // reuses the row-pass partial buffers the side-stream record reads)
    const bool ver = c0->ver_hist_on || c0->ver_xs_on;
    if (ver)
        if (int rc = ver_snapshot(c0, 0, c0->Dblk[0])) return rc;
    if (c0->algo == 1)
        if (int rc = each(ctx, X, mccg_setup)) return rc;
    if (int rc = on0()) return rc;
    CK(cudaEventRecord(c0->ev_loop0, c0->stream));
    for (coopcg_gpu_ctx* c : X.s) c->rank_async = !ver;
    struct AsyncOff {
        const Exch& X;
        ~AsyncOff() {
            for (coopcg_gpu_ctx* c : X.s) c->rank_async = false;
        }
    } async_off{X};

    // ---- main loop, enqueued in chunks; device-side stop makes extras no-ops ----
    // No host read after setup: a stop raised by the setup coordinator turns
    // the first chunk into no-ops and its snapshot ends the loop (mccg reads
    // the control block in mccg_setup already).  Every shard holds the same
    // control state (replicated), so shard 0's snapshot decides.
    bool stopped = false;
    int k_host = 0;
    int chunk_id = 0;
    double mv_total = 0.0;
    int mv_count = 0;
    int chunk_iters[2] = {0, 0};
    double trend_rate = 1.0, trend_last = 0.0;
    int trend_k = -1;
    bool chunk_rec[2][kChunkMax] = {};
    // A.D launch timing (coopcg_timing, the bench roofline): CUDA events around
    // every mv_every-th A.D of shard 0 only -- an event between two kernels
    // costs the programmatic-launch overlap there (+1.3% exact / +2.4% fast it/s
    // at cfg 2 with 8 vs 1, tools/mv_events_ab.sh).  COOPCG_MV_EVERY overrides
    // (0 = off).
    static const int mv_every = [] {
        const char* e = std::getenv("COOPCG_MV_EVERY");
        return e ? std::atoi(e) : 8;
    }();
    int chunk_k0[2] = {0, 0};
    int pending[2];
    int npending = 0;
    auto read_chunk = [&](int c) -> int {
        const int slot = c & 1;
        CK(cudaEventSynchronize(c0->ev_chunk[slot]));
        const Ctl& snap = c0->ctl_host[slot];
        for (int u = 0; u < chunk_iters[slot]; ++u) {
            const int kk = chunk_k0[slot] + u;
            if (kk >= snap.iterations) break;  // launches after the stop were no-ops
            if (!chunk_rec[slot][u]) continue;
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, c0->mv_ev[(slot * kChunkMax + u) * 2],
                                     c0->mv_ev[(slot * kChunkMax + u) * 2 + 1]) == cudaSuccess) {
                mv_total += ms;
                ++mv_count;
            }
        }
        if (snap.stop) stopped = true;
        // residual trend of the chunk (recorded minres), for sizing what to enqueue next
        const int n_done = std::min(chunk_iters[slot], snap.iterations - chunk_k0[slot]);
        if (n_done >= 2 && chunk_k0[slot] + n_done <= c0->tr_capacity) {
            const double first = c0->minres_host[slot * kChunkMax];
            trend_last = c0->minres_host[slot * kChunkMax + n_done - 1];
            // geometric-mean decay per iteration over the chunk
            trend_rate = (first > 0.0 && trend_last > 0.0) ? std::pow(trend_last / first, 1.0 / (n_done - 1)) : 1.0;
            trend_k = chunk_k0[slot] + n_done - 1;
        }
        return COOPCG_OK;
    };
    // Enqueue sizing: chunks of 4, 4, 8, 8, 16, 16, ... iterations, two in flight.
    // With a tolerance, the next chunk is capped by the iterations the recent
    // geometric decay of minres still needs (no-op launches after the stop are
    // cheap but not free: they dominated small solves such as config 0).
    // Sizing never changes results: the device stop flag decides.
    int chunk = 4, same = 0;
    for (;;) {
      while (!stopped && k_host < max_iters) {
        if (npending == 2) {
            if (int rc = read_chunk(pending[0])) return rc;
            pending[0] = pending[1];
            npending = 1;
            if (stopped) break;
        }
        const int slot = chunk_id & 1;
        int U = std::min(chunk, max_iters - k_host);
        const double tol = c0->ctl_host[0].tol;
        if (tol > 0.0 && trend_k >= 0 && trend_last > tol && trend_rate > 0.0 && trend_rate < 0.9) {
            // clear geometric convergence: enqueue about what is still needed
            const double need = std::ceil(std::log(tol / trend_last) / std::log(trend_rate));
            const int queued = k_host - (trend_k + 1);  // already enqueued beyond the last read
            const int cap = static_cast<int>(std::max(2.0, need - queued + 1.0));
            U = std::max(1, std::min(U, cap));
        }
        chunk_iters[slot] = U;
        chunk_k0[slot] = k_host;
        for (int u = 0; u < U; ++u, ++k_host) {
            const bool rec = mv_every > 0 && k_host % mv_every == 0;
            chunk_rec[slot][u] = rec;
            const int k = k_host;
            if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) {
                    const bool r = rec && c == c0;
                    return iter_local(c, k, r ? c->mv_ev[(slot * kChunkMax + u) * 2] : nullptr,
                                      r ? c->mv_ev[(slot * kChunkMax + u) * 2 + 1] : nullptr);
                }))
                return rc;
            if (int rc = xq(ctx, X, k)) return rc;
            if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return iter_mid(c, k); })) return rc;
            if (recompute_at(c0, k))
                if (int rc = xrows(ctx, X, COOPCG_BLOCK_R, k)) return rc;
            if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return iter_rest(c, k); })) return rc;
            if (ver) {
                if (int rc = ver_anorm(c0, k)) return rc;
                if (int rc = ver_snapshot(c0, k + 1, c0->Dblk[(k + 1) & 1])) return rc;
            }
        }
        if (int rc = each(ctx, X, join_rank)) return rc;
        if (int rc = on0()) return rc;
        CK(cudaMemcpyAsync(&c0->ctl_host[slot], c0->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c0->stream));
        if (chunk_k0[slot] + U <= c0->tr_capacity)
            CK(cudaMemcpyAsync(c0->minres_host + slot * kChunkMax, c0->tr_minres + chunk_k0[slot],
                               sizeof(double) * U, cudaMemcpyDeviceToHost, c0->stream));
        CK(cudaEventRecord(c0->ev_chunk[slot], c0->stream));
        pending[npending++] = chunk_id;
        ++chunk_id;
        if (++same == 2) {
            chunk = std::min(kChunkMax, chunk * 2);
            same = 0;
        }
      }
      for (int q = 0; q < npending; ++q)
          if (int rc = read_chunk(pending[q])) return rc;
      npending = 0;
      // mccg: the device paused on a rank drop (restrict_pending); every shard
      // holds the same replicated blocks and takes the same decision.
      if (c0->algo != 1) break;
      if (int rc = on0()) return rc;
      CK(cudaMemcpyAsync(&c0->ctl_host[0], c0->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c0->stream));
      CK(cudaStreamSynchronize(c0->stream));
      if (!c0->ctl_host[0].restrict_pending) break;
      const int kr = c0->ctl_host[0].k;
      int next_k = -1;
      if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return mccg_restrict(c, kr, &next_k); })) return rc;
      if (next_k < 0) break;
      k_host = next_k;
      stopped = false;
      chunk = 4;
      same = 0;
      trend_k = -1;
    }
    if (int rc = each(ctx, X, join_rank)) return rc;
    for (coopcg_gpu_ctx* c : X.s) c->rank_async = false;
    if (int rc = on0()) return rc;
    CK(cudaEventRecord(c0->ev_loop1, c0->stream));
    if (int rc = each(ctx, X, final_local)) return rc;
    if (int rc = xrows(ctx, X, COOPCG_BLOCK_S, 0)) return rc;
    if (int rc = each(ctx, X, final_rest)) return rc;
    if (int rc = xbarrier(ctx, X)) return rc;  // shard 0's end event after every shard's work
    if (int rc = on0()) return rc;
    CK(cudaEventRecord(c0->ev_run1, c0->stream));
    if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) -> int {
            cudaError_t e = cudaStreamSynchronize(c->stream);
            return e == cudaSuccess ? COOPCG_OK
                                    : fail(c, COOPCG_E_CUDA, "stream synchronize: %s", cudaGetErrorString(e));
        }))
        return rc;
    if (int rc = on0()) return rc;
    float run_ms = 0.f, loop_ms = 0.f;
    CK(cudaEventElapsedTime(&run_ms, c0->ev_run0, c0->ev_run1));
    CK(cudaEventElapsedTime(&loop_ms, c0->ev_loop0, c0->ev_loop1));
    long long launches = 0;
    for (coopcg_gpu_ctx* c : X.s) launches += c->launches;
    coopcg_timing tm{};
    tm.run_ms = run_ms;
    tm.loop_ms = loop_ms;
    tm.matvec_ms_total = mv_total;
    tm.matvec_launches = mv_count;
    tm.kernel_launches = launches;
    c0->timing = tm;
    ctx->timing = tm;
    if (guard_enabled())
        for (coopcg_gpu_ctx* c : X.s) {
            std::string what;
            if (check_guards(c, what)) return fail(ctx, COOPCG_E_CUDA, "COOPCG_GUARD: %s", what.c_str());
        }
    const int rc = end_impl(c0, trace);
    if (rc != COOPCG_OK && c0 != ctx) ctx->msg = c0->msg;
    return rc;
}

extern "C" {

int coopcg_gpu_run(coopcg_gpu_ctx* ctx, const coopcg_opts* opts, coopcg_trace* trace) {
    if (!ctx) return COOPCG_E_INVALID;
    if (!is_group(ctx)) CK(cudaSetDevice(ctx->device));
    return run_impl(ctx, opts, trace);
}

int coopcg_gpu_begin(coopcg_gpu_ctx* ctx, const coopcg_opts* opts) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    if (ctx->ver_hist_on || ctx->ver_xs_on)
        return fail(ctx, COOPCG_E_INVALID, "verification mode (keep_history / x_star) runs whole solves (coopcg_gpu_run)");
    CK(cudaSetDevice(ctx->device));
    return begin_impl(ctx, opts);
}

int coopcg_gpu_phase(coopcg_gpu_ctx* ctx, int phase, int k) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    switch (phase) {
    case COOPCG_PH_SETUP_LOCAL: return setup_local(ctx);
    case COOPCG_PH_SETUP_REST: return setup_rest(ctx);
    case COOPCG_PH_ITER_LOCAL: {
        // A.D launch timing for the phase-driven (sharded) solve: events around
        // every 8th A.D, the first kChunkMax of them (read by coopcg_gpu_end)
        const bool rec = k % 8 == 0 && ctx->phase_mv < kChunkMax;
        cudaEvent_t e0 = rec ? ctx->mv_ev[ctx->phase_mv * 2] : nullptr;
        cudaEvent_t e1 = rec ? ctx->mv_ev[ctx->phase_mv * 2 + 1] : nullptr;
        if (rec) ++ctx->phase_mv;
        return iter_local(ctx, k, e0, e1);
    }
    case COOPCG_PH_ITER_MID: return iter_mid(ctx, k);
    case COOPCG_PH_ITER_REST: return iter_rest(ctx, k);
    case COOPCG_PH_FINAL_LOCAL: return final_local(ctx);
    case COOPCG_PH_FINAL_REST: return final_rest(ctx);
    case COOPCG_PH_MCCG_SETUP: return ctx->algo == 1 ? mccg_setup(ctx) : COOPCG_OK;
    default: return fail(ctx, COOPCG_E_INVALID, "unknown phase %d", phase);
    }
}

int coopcg_gpu_mccg_resume(coopcg_gpu_ctx* ctx, int* next_k) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx || !next_k) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    *next_k = -1;
    if (ctx->algo != 1) return COOPCG_OK;
    CK(cudaMemcpyAsync(&ctx->ctl_host[0], ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (!ctx->ctl_host[0].restrict_pending) return COOPCG_OK;
    return mccg_restrict(ctx, ctx->ctl_host[0].k, next_k);
}

int coopcg_gpu_recompute_at(const coopcg_gpu_ctx* ctx, int k) {
    if (is_group(ctx)) ctx = ctx->shards[0];
    return ctx ? (recompute_at(ctx, k) ? 1 : 0) : 0;
}

int coopcg_gpu_ipc_handles(coopcg_gpu_ctx* ctx, void* handles_out) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx || !handles_out) return COOPCG_E_INVALID;
    if (!sharded(ctx)) return fail(ctx, COOPCG_E_STATE, "peer exchange is for row-sharded contexts");
    if (guard_enabled())
        return fail(ctx, COOPCG_E_STATE, "CUDA IPC exchange is unavailable with COOPCG_GUARD=1 (guarded buffers)");
    CK(cudaSetDevice(ctx->device));
    if (!ctx->Qalt) {
        CK(cudaMalloc(&ctx->Qalt, sizeof(double) * (size_t)ctx->n * ctx->P));
        CK(cudaMemset(ctx->Qalt, 0, sizeof(double) * (size_t)ctx->n * ctx->P));
    }
    double* bufs[2] = {ctx->Q, ctx->Qalt};
    for (int b = 0; b < 2; ++b) {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, bufs[b]));
        std::memcpy(static_cast<char*>(handles_out) + b * COOPCG_IPC_HANDLE_BYTES, &h, COOPCG_IPC_HANDLE_BYTES);
    }
    return COOPCG_OK;
}

int coopcg_gpu_set_peers(coopcg_gpu_ctx* ctx, int nranks, int self_rank, const void* handles) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx || !handles) return COOPCG_E_INVALID;
    if (nranks < 1 || nranks > kMaxPeers || self_rank < 0 || self_rank >= nranks)
        return fail(ctx, COOPCG_E_INVALID, "set_peers: nranks %d (max %d), self %d", nranks, kMaxPeers, self_rank);
    if (!ctx->Qalt) return fail(ctx, COOPCG_E_STATE, "set_peers: call coopcg_gpu_ipc_handles first");
    CK(cudaSetDevice(ctx->device));
    static_assert(sizeof(cudaIpcMemHandle_t) == COOPCG_IPC_HANDLE_BYTES, "IPC handle size");
    double* own[2] = {ctx->Q, ctx->Qalt};
    PeerRows pr[2] = {};
    for (int r = 0; r < nranks; ++r)
        for (int b = 0; b < 2; ++b) {
            if (r == self_rank) {
                pr[b].dst[r] = own[b];
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + (r * 2 + b) * COOPCG_IPC_HANDLE_BYTES,
                        COOPCG_IPC_HANDLE_BYTES);
            void* ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_opened.push_back(ptr);
            pr[b].dst[r] = static_cast<double*>(ptr);
        }
    pr[0].n = pr[1].n = nranks;
    ctx->peers[0] = pr[0];
    ctx->peers[1] = pr[1];
    ctx->p2p = true;
    return COOPCG_OK;
}

int coopcg_gpu_block(coopcg_gpu_ctx* ctx, int which, int k, void** dev_ptr, int* ld) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx || !dev_ptr) return COOPCG_E_INVALID;
    double* b = nullptr;
    switch (which) {
    case COOPCG_BLOCK_X: b = ctx->X; break;
    case COOPCG_BLOCK_R: b = ctx->R; break;
    case COOPCG_BLOCK_D: b = ctx->Dblk[k & 1]; break;
    case COOPCG_BLOCK_Q: b = q_of(ctx, k); break;
    case COOPCG_BLOCK_S: b = ctx->S; break;
    case COOPCG_BLOCK_W:
        if (!ctx->hh_w) return fail(ctx, COOPCG_E_STATE, "no Householder generation in progress");
        *dev_ptr = ctx->hh_w;
        if (ld) *ld = 1;
        return COOPCG_OK;
    default: return fail(ctx, COOPCG_E_INVALID, "unknown block %d", which);
    }
    *dev_ptr = b;
    if (ld) *ld = ctx->P;
    return COOPCG_OK;
}

int coopcg_gpu_state(coopcg_gpu_ctx* ctx, int* stop, int* iterations) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(&ctx->ctl_host[1], ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (stop) *stop = ctx->ctl_host[1].stop;
    if (iterations) *iterations = ctx->ctl_host[1].iterations;
    return COOPCG_OK;
}

int coopcg_gpu_end(coopcg_gpu_ctx* ctx, coopcg_trace* trace) {
    if (is_group(ctx))
        return fail(ctx, COOPCG_E_STATE, "a multi-device handle runs whole solves (coopcg_gpu_run / _solve)");
    if (!ctx) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    ctx->timing.kernel_launches = ctx->launches;
    const int rc = end_impl(ctx, trace);  // synchronises the stream
    if (rc == COOPCG_OK && guard_enabled()) {
        std::string what;
        if (check_guards(ctx, what)) return fail(ctx, COOPCG_E_CUDA, "COOPCG_GUARD: %s", what.c_str());
    }
    if (rc != COOPCG_OK) return rc;
    // the phase API's sampled A.D launches (iteration 8 i; later ones were no-ops)
    double tot = 0.0;
    int cnt = 0;
    for (int i = 0; i < ctx->phase_mv && 8 * i < ctx->ctl_host[0].iterations; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ctx->mv_ev[2 * i], ctx->mv_ev[2 * i + 1]) == cudaSuccess) {
            tot += ms;
            ++cnt;
        }
    }
    ctx->timing.matvec_ms_total = tot;
    ctx->timing.matvec_launches = cnt;
    return COOPCG_OK;
}

int coopcg_gpu_solve(coopcg_gpu_ctx* ctx, const double* b, const double* X0, const coopcg_opts* opts,
                     coopcg_trace* trace) {
    if (int rc = coopcg_gpu_upload(ctx, b, X0)) return rc;
    return coopcg_gpu_run(ctx, opts, trace);
}

int coopcg_gpu_set_verification(coopcg_gpu_ctx* ctx, int keep_history, const double* x_star) {
    if (!ctx) return COOPCG_E_INVALID;
    if ((keep_history || x_star) && (is_group(ctx) || sharded(ctx) || ctx->nccl))
        return fail(ctx, COOPCG_E_INVALID,
                    "verification mode (keep_history / x_star) needs one context holding every row of A");
    CK(cudaSetDevice(ctx->device));
    ctx->ver_hist_on = keep_history != 0;
    ctx->ver_xs_on = x_star != nullptr;
    ctx->ver_iters = -1;
    if (x_star) {
        if (!ctx->ver_xs) CK(gmalloc(ctx, &ctx->ver_xs, sizeof(double) * (size_t)ctx->n, "ver_xs"));
        CK(cudaMemcpyAsync(ctx->ver_xs, x_star, sizeof(double) * (size_t)ctx->n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return COOPCG_OK;
}

int coopcg_gpu_history_count(const coopcg_gpu_ctx* ctx, int* entries) {
    if (!ctx || !entries) return COOPCG_E_INVALID;
    *entries = (ctx->ver_hist_on && ctx->ver_iters >= 0) ? ctx->ver_iters + 1 : 0;
    return COOPCG_OK;
}

int coopcg_gpu_get_history(coopcg_gpu_ctx* ctx, int entry, double* X, double* R, double* D) {
    if (!ctx) return COOPCG_E_INVALID;
    if (!ctx->ver_hist_on || ctx->ver_iters < 0)
        return fail(ctx, COOPCG_E_STATE, "no history: run a solve after coopcg_gpu_set_verification(ctx, 1, ...)");
    if (entry < 0 || entry > ctx->ver_iters || entry >= ctx->ver_hist_cap)
        return fail(ctx, COOPCG_E_INVALID, "history entry %d outside [0, %d]", entry, ctx->ver_iters);
    CK(cudaSetDevice(ctx->device));
    const int n = ctx->n, p = ctx->p_orig, P = ctx->P;
    const size_t blk = (size_t)n * P;
    double* outs[3] = {X, R, D};
    for (int b = 0; b < 3; ++b) {
        if (!outs[b]) continue;
        rowmajor_to_colmajor_kernel<<<grid_for((size_t)n * p, 256), 256, 0, ctx->stream>>>(
            ctx->ver_hist + ((size_t)entry * 3 + b) * blk, ctx->stage, n, p, P);
        CKL();
        CK(cudaMemcpyAsync(outs[b], ctx->stage, sizeof(double) * (size_t)n * p, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return COOPCG_OK;
}

int coopcg_gpu_get_anorm_errors(coopcg_gpu_ctx* ctx, int capacity, double* out) {
    if (!ctx || !out) return COOPCG_E_INVALID;
    if (!ctx->ver_xs_on || ctx->ver_iters < 0)
        return fail(ctx, COOPCG_E_STATE, "no A-norm errors: run a solve after coopcg_gpu_set_verification(ctx, ., x_star)");
    const int rows = std::min({capacity, ctx->ver_iters, ctx->ver_anorm_cap});
    if (rows <= 0) return COOPCG_OK;
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(out, ctx->ver_anorm, sizeof(double) * (size_t)rows * ctx->p_orig, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return COOPCG_OK;
}

int coopcg_gpu_timing(const coopcg_gpu_ctx* ctx, coopcg_timing* out) {
    if (!ctx || !out) return COOPCG_E_INVALID;
    *out = ctx->timing;
    out->a_l2_resident_bytes = (double)ctx->res_bytes;
    for (const coopcg_gpu_ctx* c : ctx->shards) out->a_l2_resident_bytes += (double)c->res_bytes;
    return COOPCG_OK;
}

void* coopcg_gpu_stream(const coopcg_gpu_ctx* ctx) {
    if (is_group(ctx)) return (void*)ctx->shards[0]->stream;
    return ctx ? (void*)ctx->stream : nullptr;
}

int coopcg_gpu_matvec_block(coopcg_gpu_ctx* ctx, const double* D, double* out) {
    if (is_group(ctx)) return (D && out) ? group_matvec_block(ctx, D, out) : COOPCG_E_INVALID;
    if (!ctx || !D || !out) return COOPCG_E_INVALID;
    if (!ctx->a_ready) return fail(ctx, COOPCG_E_STATE, "A not set");
    CK(cudaSetDevice(ctx->device));
    if (ctx->p != ctx->p_orig)
        if (int rc = set_active_p(ctx, ctx->p_orig)) return rc;
    const int n = ctx->n, p = ctx->p, P = ctx->P;
    cudaStream_t st = ctx->stream;
    CK(cudaMemcpyAsync(ctx->stage, D, sizeof(double) * (size_t)n * p, cudaMemcpyHostToDevice, st));
    colmajor_to_rowmajor_kernel<<<grid_for((size_t)n * P, 256), 256, 0, st>>>(ctx->stage, ctx->Dblk[0], n, p, P);
    CKL();
    if (ctx->arith == COOPCG_ARITH_FAST) {
        CK(fast_ad(ctx, ctx->Dblk[0], nullptr));
        CK(fast_rows(ctx, ctx->Q, nullptr, nullptr, nullptr, nullptr, 1, nullptr));
    } else {
        CK(ad_launch(ctx, ctx->Dblk[0], ctx->Q, nullptr, nullptr));
    }
    rowmajor_to_colmajor_kernel<<<grid_for((size_t)ctx->n_loc * p, 256), 256, 0, st>>>(
        ctx->Q + (size_t)ctx->row0 * P, ctx->stage, ctx->n_loc, p, P);
    CKL();
    CK(cudaMemcpyAsync(out, ctx->stage, sizeof(double) * (size_t)ctx->n_loc * p, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return COOPCG_OK;
}

int coopcg_gpu_numerical_rank_ex(coopcg_gpu_ctx* ctx, const double* D, double tol, int force_exact, int* rank) {
    if (is_group(ctx)) return coopcg_gpu_numerical_rank_ex(ctx->shards[0], D, tol, force_exact, rank);
    if (!ctx || !D || !rank) return COOPCG_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    if (ctx->p != ctx->p_orig)
        if (int rc = set_active_p(ctx, ctx->p_orig)) return rc;
    const int n = ctx->n, p = ctx->p, P = ctx->P;
    cudaStream_t st = ctx->stream;
    Ctl h{};
    h.p = p;
    h.P = P;
    h.rank_rel_tol = tol;
    h.max_iters = 1;
    h.force_exact = force_exact;
    std::memcpy(&ctx->ctl_host[0], &h, sizeof(Ctl));
    CK(cudaMemcpyAsync(ctx->ctl, &ctx->ctl_host[0], sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->stage, D, sizeof(double) * (size_t)n * p, cudaMemcpyHostToDevice, st));
    colmajor_to_rowmajor_kernel<<<grid_for((size_t)n * P, 256), 256, 0, st>>>(ctx->stage, ctx->Dblk[1], n, p, P);
    CKL();
    const int dgrid = exact_dgrid(ctx);
    CK(gram_partials_launch(ctx, ctx->Dblk[1], dgrid, nullptr));
    rank_end_kernel<<<1, 1024, rank_smem(P), st>>>(ctx->partials, dgrid, ctx->Dblk[1], ctx->V, n, ctx->ctl, 2, nullptr);
    CKL();
    CK(cudaMemcpyAsync(&ctx->ctl_host[0], ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *rank = ctx->ctl_host[0].rank_result;
    return COOPCG_OK;
}

int coopcg_gpu_numerical_rank(coopcg_gpu_ctx* ctx, const double* D, double tol, int* rank) {
    return coopcg_gpu_numerical_rank_ex(ctx, D, tol, 0, rank);
}

}  // extern "C"

// =============================================================================
// Multi-GPU contexts: a group handle over in-process row shards
// and rank contexts with NCCL row exchanges.
// =============================================================================
static int group_set_A(coopcg_gpu_ctx* ctx, const double* A_rows) {
    const Exch X = exch_of(ctx);
    return each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_set_A(c, A_rows + (size_t)c->row0 * c->n); });
}

static int group_get_A_rows(coopcg_gpu_ctx* ctx, int row0, int rows, double* A_rows) {
    if (row0 < 0 || rows < 0 || row0 + rows > ctx->n)
        return fail(ctx, COOPCG_E_DIMENSION, "get_A_rows: row range outside the matrix");
    const Exch X = exch_of(ctx);
    return each(ctx, X, [&](coopcg_gpu_ctx* c) {
        const int a = std::max(row0, c->row0), b = std::min(row0 + rows, c->row1);
        if (a >= b) return (int)COOPCG_OK;
        return coopcg_gpu_get_A_rows(c, a - c->row0, b - a, A_rows + (size_t)(a - row0) * c->n);
    });
}

// The Householder generator over row shards: each shard computes its rows of
// w = M v, the rows are exchanged, every shard forms the scalars from the full
// vectors identically and updates its rows.
static int gen_householder_x(coopcg_gpu_ctx* ctx, const Exch& X, uint64_t seed, int m, double kappa) {
    for (coopcg_gpu_ctx* c : X.s) c->a_ready = false;
    if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_gen_householder_begin(c, seed, m, kappa); }))
        return rc;
    for (int r = m - 1; r >= 0; --r) {
        if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_gen_householder_local(c, r); }))
            return rc;
        if (int rc = xrows(ctx, X, COOPCG_BLOCK_W, 0)) return rc;
        if (int rc = each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_gen_householder_rest(c, r); }))
            return rc;
    }
    return each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_gen_householder_end(c); });
}

static int rank_gen_householder(coopcg_gpu_ctx* ctx, uint64_t seed, int m, double kappa) {
    return gen_householder_x(ctx, exch_of(ctx), seed, m, kappa);
}

static int group_gen_A(coopcg_gpu_ctx* ctx, int kind, uint64_t seed, int m, double kappa) {
    const Exch X = exch_of(ctx);
    if (kind == COOPCG_MATRIX_DIAGDOM)
        return each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_gen_A(c, kind, seed, m, kappa); });
    if (kind == COOPCG_MATRIX_HOUSEHOLDER) return gen_householder_x(ctx, X, seed, m, kappa);
    return fail(ctx, COOPCG_E_INVALID, "matrix kind %d needs the whole matrix on one device", kind);
}

static int group_upload(coopcg_gpu_ctx* ctx, const double* b, const double* X0) {
    const Exch X = exch_of(ctx);
    return each(ctx, X, [&](coopcg_gpu_ctx* c) { return coopcg_gpu_upload(c, b, X0); });
}

static int group_matvec_block(coopcg_gpu_ctx* ctx, const double* D, double* out) {
    const Exch X = exch_of(ctx);
    const int n = ctx->n, p = ctx->p_orig;
    std::vector<double> part;
    return each(ctx, X, [&](coopcg_gpu_ctx* c) {
        part.resize((size_t)c->n_loc * p);
        if (int rc = coopcg_gpu_matvec_block(c, D, part.data())) return rc;
        for (int j = 0; j < p; ++j)  // column-major n_loc x p -> rows [row0, row1) of the n x p output
            std::memcpy(out + (size_t)j * n + c->row0, part.data() + (size_t)j * c->n_loc, sizeof(double) * c->n_loc);
        return (int)COOPCG_OK;
    });
}

extern "C" {

int coopcg_row_split(int n, int parts, int part, int* row_begin, int* row_end) {
    if (n < 1 || parts < 1 || part < 0 || part >= parts || !row_begin || !row_end) return COOPCG_E_INVALID;
    row_split(n, parts, part, row_begin, row_end);
    return COOPCG_OK;
}

int coopcg_gpu_create_multi(int n, int p, int ndev, const int* devices, int arith, coopcg_gpu_ctx** out) {
    if (!out || !devices || ndev < 1) return COOPCG_E_INVALID;
    *out = nullptr;
    g_create_error.clear();
    if (ndev > kMaxPeers) return fail(nullptr, COOPCG_E_INVALID, "ndev %d > %d", ndev, kMaxPeers);
    if (ndev == 1) return coopcg_gpu_create(n, p, devices[0], arith, out);
    for (int g = 0; g < ndev; ++g) {
        int r0 = 0, r1 = 0;
        row_split(n, ndev, g, &r0, &r1);
        if (r1 <= r0) return fail(nullptr, COOPCG_E_DIMENSION, "n = %d rows cannot be split over %d devices", n, ndev);
    }
    auto* ctx = new coopcg_gpu_ctx();
    ctx->n = n;
    ctx->p = ctx->p_orig = p;
    ctx->device = devices[0];
    ctx->arith = arith;
    ctx->row0 = 0;
    ctx->row1 = ctx->n_loc = n;
    auto bail = [&](int code) {
        const std::string m = ctx->msg.empty() ? g_create_error : ctx->msg;
        destroy_impl(ctx);
        g_create_error = m;
        return code;
    };
    for (int g = 0; g < ndev; ++g) {
        int r0 = 0, r1 = 0;
        row_split(n, ndev, g, &r0, &r1);
        coopcg_gpu_ctx* c = nullptr;
        if (int rc = coopcg_gpu_create_shard(n, p, devices[g], arith, r0, r1, &c)) return bail(rc);
        ctx->shards.push_back(c);
    }
    for (int g = 0; g < ndev; ++g)  // shards sharing a device share its L2
        set_l2_residency(ctx->shards[g], (int)std::count(devices, devices + ndev, devices[g]));
    ctx->P = ctx->shards[0]->P;
    // peer access between distinct devices (the Q rows are stored straight
    // into every shard's Q by the kernel that computes them)
    for (int g = 0; g < ndev; ++g)
        for (int h = 0; h < ndev; ++h) {
            if (devices[g] == devices[h]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, devices[g], devices[h]);
            if (!can) {
                fail(ctx, COOPCG_E_CUDA, "device %d cannot access device %d (peer access)", devices[g], devices[h]);
                return bail(COOPCG_E_CUDA);
            }
            cudaSetDevice(devices[g]);
            cudaError_t e = cudaDeviceEnablePeerAccess(devices[h], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else if (e != cudaSuccess) {
                fail(ctx, COOPCG_E_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", devices[g], devices[h],
                     cudaGetErrorString(e));
                return bail(COOPCG_E_CUDA);
            }
        }
    // Q double-buffered by iteration parity (a shard pushing iteration k+1
    // never overwrites rows a slower shard still reads in k)
    for (coopcg_gpu_ctx* c : ctx->shards) {
        cudaSetDevice(c->device);
        const size_t bytes = sizeof(double) * (size_t)n * c->P;
        if (gmalloc(c, &c->Qalt, bytes, "Q (odd iterations)") != cudaSuccess ||
            cudaMemset(c->Qalt, 0, bytes) != cudaSuccess) {
            fail(ctx, COOPCG_E_CUDA, "allocating the second Q buffer on device %d", c->device);
            return bail(COOPCG_E_CUDA);
        }
    }
    for (coopcg_gpu_ctx* c : ctx->shards) {
        PeerRows pr[2] = {};
        for (int h = 0; h < ndev; ++h) {
            pr[0].dst[h] = ctx->shards[h]->Q;
            pr[1].dst[h] = ctx->shards[h]->Qalt;
        }
        pr[0].n = pr[1].n = ndev;
        c->peers[0] = pr[0];
        c->peers[1] = pr[1];
        c->p2p = true;
    }
    ctx->gev.assign(ndev, nullptr);
    for (int g = 0; g < ndev; ++g) {
        cudaSetDevice(devices[g]);
        if (cudaEventCreateWithFlags(&ctx->gev[g], cudaEventDisableTiming) != cudaSuccess) {
            fail(ctx, COOPCG_E_CUDA, "event creation on device %d", devices[g]);
            return bail(COOPCG_E_CUDA);
        }
    }
    cudaSetDevice(devices[0]);
    *out = ctx;
    return COOPCG_OK;
}

int coopcg_nccl_unique_id(void* id_out) {
    if (!id_out) return COOPCG_E_INVALID;
    const NcclApi& api = nccl_api();
    if (!api.getUniqueId) return fail(nullptr, COOPCG_E_CUDA, "NCCL unavailable: %s", api.err.c_str());
    static_assert(sizeof(ncclUniqueId) == COOPCG_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = api.getUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, COOPCG_E_CUDA, "ncclGetUniqueId: %s", nccl_err(r));
    std::memcpy(id_out, &id, sizeof id);
    return COOPCG_OK;
}

int coopcg_gpu_create_rank(int n, int p, int device, int arith, int nranks, int rank, const void* nccl_id,
                           coopcg_gpu_ctx** out) {
    if (!out || !nccl_id || nranks < 1 || rank < 0 || rank >= nranks) return COOPCG_E_INVALID;
    *out = nullptr;
    int r0 = 0, r1 = 0;
    row_split(n, nranks, rank, &r0, &r1);
    if (r1 <= r0) return fail(nullptr, COOPCG_E_DIMENSION, "n = %d rows cannot be split over %d ranks", n, nranks);
    const NcclApi& api = nccl_api();
    if (!api.getUniqueId) return fail(nullptr, COOPCG_E_CUDA, "NCCL unavailable: %s", api.err.c_str());
    coopcg_gpu_ctx* ctx = nullptr;
    if (int rc = coopcg_gpu_create_shard(n, p, device, arith, r0, r1, &ctx)) return rc;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    ncclComm_t comm = nullptr;
    cudaSetDevice(device);
    ncclResult_t r = api.commInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
        destroy_impl(ctx);
        return fail(nullptr, COOPCG_E_CUDA, "ncclCommInitRank(%d of %d): %s", rank, nranks, nccl_err(r));
    }
    ctx->nccl = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    *out = ctx;
    return COOPCG_OK;
}

int coopcg_gpu_shards(const coopcg_gpu_ctx* ctx, int cap, int* nshards, int* devices, int* row_begin, int* row_end) {
    if (!ctx || !nshards) return COOPCG_E_INVALID;
    const int ns = is_group(ctx) ? (int)ctx->shards.size() : 1;
    *nshards = ns;
    for (int g = 0; g < ns && g < cap; ++g) {
        const coopcg_gpu_ctx* c = is_group(ctx) ? ctx->shards[g] : ctx;
        if (devices) devices[g] = c->device;
        if (row_begin) row_begin[g] = c->row0;
        if (row_end) row_end[g] = c->row1;
    }
    return COOPCG_OK;
}

}  // extern "C"
