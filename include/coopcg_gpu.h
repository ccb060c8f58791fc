/*
 * coopcg_gpu.h -- C ABI of the B200-native cooperative-CG hot path.
 *
 * Drop-in boundary for the reference's solver entry point
 *   template<ScalarField S> SolveTrace<S> ccg_solve(const SpdMatrix<S>&,
 *       const Vec<S>&, const DenseBlock<S>&, const SolveOptions<S>& = {})
 *   (/root/reference/proj/include/coopcg/solvers.hpp:329-333)
 * and its OpenMP twin parallel_ccg (coopcg/parallel.hpp:76-111).  The
 * reference's executor policy (drive<S,Exec>, solvers.hpp:259-262) is per-slot
 * and host-memory based, so the GPU backend plugs in at solver level: the C++
 * header include/coopcg/gpu_ccg.hpp wraps these functions into
 *   coopcg::gpu_ccg(A, b, X0, opts, gpu_opts) -> SolveTrace<double>
 * with ccg_solve's semantics; INTEGRATION.md shows the binding.
 *
 * No C++ or torch types cross this boundary: plain pointers, sizes, PODs.
 * Every function returns an int code (coopcg_err); the context keeps the last
 * message (coopcg_gpu_last_error).  Contexts are independent: no global
 * mutable state, one CUDA stream per context (reentrant per context, like the
 * reference's concurrent independent solves, tests/test_parallel.cpp:190-204).
 *
 * Layouts at the boundary are the reference's: A row-major n x n
 * (coopcg/dense.hpp:101-170); X0 / final_x column-major n x p DenseBlock
 * (dense.hpp:35-38).  Device layouts are private.
 */
#ifndef COOPCG_GPU_H
#define COOPCG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COOPCG_GPU_ABI_VERSION 2 /* 2: verification mode (set_verification, get_history, get_anorm_errors) */
#define COOPCG_GPU_MAX_P 32

/* Error codes; map to the reference exception hierarchy (errors.hpp:11-41). */
enum coopcg_err {
    COOPCG_OK = 0,
    COOPCG_E_DIMENSION = 1,            /* DimensionError */
    COOPCG_E_SPD_VIOLATION = 2,        /* SpdViolationError */
    COOPCG_E_NUMERICAL_BREAKDOWN = 3,  /* NumericalBreakdownError */
    COOPCG_E_SINGULAR = 4,             /* SingularMatrixError */
    COOPCG_E_INVALID = 5,              /* bad argument (null pointer, bad enum) */
    COOPCG_E_STATE = 6,                /* call out of order (e.g. run before A set) */
    COOPCG_E_CUDA = 10                 /* CUDA runtime error; message has details */
};

/* TerminalStatus (trace.hpp:13-17). */
enum coopcg_status {
    COOPCG_CONVERGED = 0,
    COOPCG_RANK_COLLAPSE = 1,
    COOPCG_MAX_ITERATIONS = 2
};

/* Arithmetic modes.  EXACT reproduces the reference's
 * floating-point operation order bit for bit; FAST reorders (DFMA/DMMA,
 * tree reductions, Cholesky) for the roofline. */
enum coopcg_arith { COOPCG_ARITH_EXACT = 0, COOPCG_ARITH_FAST = 1 };

/* On-device matrix generators.  RANDOM_SPD is the reference's
 * own generator random_spd(n, cond = kappa, seed) (problem.hpp:118-152:
 * Haar-orthogonal U by modified Gram-Schmidt, A = (U Lambda) U^T, SpdMatrix
 * symmetrisation), bit-identical to it (m is ignored). */
enum coopcg_matrix_kind { COOPCG_MATRIX_DIAGDOM = 0, COOPCG_MATRIX_HOUSEHOLDER = 1, COOPCG_MATRIX_RANDOM_SPD = 2 };
enum coopcg_vector_kind { COOPCG_VEC_UNIFORM = 0, COOPCG_VEC_NORMAL = 1 };

/* SolveOptions<double> (trace.hpp:74-88).  The verification-only fields
 * keep_history / x_star are set per context with coopcg_gpu_set_verification. */
typedef struct {
    double tol;                   /* absolute threshold on ||r_j||_2 (block_cg.hpp:283-289) */
    int max_iters;                /* -1 => 2n (solvers.hpp:18-23) */
    int recompute_residual_every; /* -1 => 50; 0 disables (solvers.hpp:25-35) */
    double rank_rel_tol;          /* numerical_rank tolerance, reference default 1e-10 */
    int algo;                     /* 0 = ccg_solve (solvers.hpp:329-333), 1 = mccg_solve (:338-342),
                                     2 = steepest_descent_solve (p = 1, exact; :532-646).
                                     cg_solve (:388-530) is algo 0 with p = 1 and
                                     recompute_residual_every defaulting to 1. */
} coopcg_opts;

/* SolveTrace<double> (trace.hpp:46-71), caller-allocated arrays.
 * Any array pointer may be NULL to skip that output. */
typedef struct {
    int capacity;                   /* rows the per-iteration arrays can hold */
    double* residual_norms;         /* [capacity * p]; row k = IterationRecord::residual_norms */
    double* minres;                 /* [capacity] */
    uint64_t* wall_ns;              /* [capacity]; device clock, per iteration */
    double* initial_residual_norms; /* [p] */
    double* final_x;                /* [n * p], column-major (DenseBlock) */
    double* final_residual_norms;   /* [p], true recomputation ||A x_j - b|| */
    /* outputs */
    int status;                     /* coopcg_status */
    int converged_agent;            /* -1 unless converged */
    int iterations;                 /* IterationRecord count */
    double initial_minres;
    double final_minres;
    uint64_t loop_wall_ns;          /* sum of wall_ns (solvers.hpp:145) */
    int exact_rank_checks;          /* diagnostics: certificate fell back to exact MGS */
    int* active_agents;             /* [p] surviving agent ids (SolveTrace::active_agents), may be NULL */
    int n_active;                   /* number of surviving agents (p unless mccg restricted) */
} coopcg_trace;
/* mccg: per-iteration norms are stored per ORIGINAL agent id (row k of
 * residual_norms has NaN for agents no longer active, IterationRecord::agents
 * = the non-NaN ids); final_x / final_residual_norms hold NaN for dropped
 * agents. */

/* Per-kernel timing of the last run, from CUDA events on the context stream. */
typedef struct {
    int matvec_launches;            /* A.D launches timed in the last run */
    double matvec_ms_total;         /* sum of their event durations */
    double run_ms;                  /* event time of the whole last run (setup..finalize) */
    double loop_ms;                 /* event time of the iteration loop only */
    long long kernel_launches;      /* kernels this library launched in the last run */
    double a_l2_resident_bytes;     /* bytes of A the A.D keeps in L2 across iterations
                                       (evict-last k-range; COOPCG_L2_RES_MB) */
} coopcg_timing;

typedef struct coopcg_gpu_ctx coopcg_gpu_ctx;

/* Library version / build information, e.g. "coopcg_gpu 1 sm_100a". */
const char* coopcg_gpu_version(void);

/* Create a context for an n x n system with p agents on CUDA `device`.
 * Owns the rows [row_begin, row_end) of A (row_begin = 0, row_end = n for a
 * single-GPU solve).  1 <= p < n, p <= COOPCG_GPU_MAX_P. */
int coopcg_gpu_create(int n, int p, int device, int arith, coopcg_gpu_ctx** out);
int coopcg_gpu_create_shard(int n, int p, int device, int arith, int row_begin, int row_end,
                            coopcg_gpu_ctx** out);
int coopcg_gpu_destroy(coopcg_gpu_ctx* ctx);

/* Copy the last error message (NUL-terminated, truncated to len).  With
 * ctx == NULL: the calling thread's last coopcg_gpu_create* failure. */
int coopcg_gpu_last_error(const coopcg_gpu_ctx* ctx, char* buf, size_t len);

/* Load this context's row block of A: rows [row_begin, row_end) of the
 * row-major n x n matrix, i.e. (row_end - row_begin) x n doubles, host memory. */
int coopcg_gpu_set_A(coopcg_gpu_ctx* ctx, const double* A_rows);
/* Generate A on the device.  DIAGDOM ignores m, kappa.
 * HOUSEHOLDER on a full context (row-sharded: the steps below). */
int coopcg_gpu_gen_A(coopcg_gpu_ctx* ctx, int kind, uint64_t seed, int m, double kappa);
/* HOUSEHOLDER generation in steps, for row-sharded contexts (each owns its
 * rows of A):
 *   begin; for r = m-1 .. 0: { local(r); <all-gather the rows of w,
 *   COOPCG_BLOCK_W>; rest(r) }; end.
 * coopcg_gpu_gen_A(HOUSEHOLDER) runs the same steps on a full context. */
int coopcg_gpu_gen_householder_begin(coopcg_gpu_ctx* ctx, uint64_t seed, int m, double kappa);
int coopcg_gpu_gen_householder_local(coopcg_gpu_ctx* ctx, int r);
int coopcg_gpu_gen_householder_rest(coopcg_gpu_ctx* ctx, int r);
int coopcg_gpu_gen_householder_end(coopcg_gpu_ctx* ctx);
/* Download this context's row block of A (row-major), for verification. */
int coopcg_gpu_get_A(coopcg_gpu_ctx* ctx, double* A_rows);
/* Rows [row0, row0 + rows) of this context's row block (row-major,
 * rows x n), e.g. to compare a 137 GB matrix with a host copy in slices. */
int coopcg_gpu_get_A_rows(coopcg_gpu_ctx* ctx, int row0, int rows, double* A_rows);

/* Host-side generators for b and X0. */
int coopcg_gen_rhs(int n, int kind, uint64_t seed, double* b);
int coopcg_gen_starts(int n, int p, uint64_t seed, double* X0_colmajor);
/* Host part of the Householder generator: reflector vectors V (m x n) and
 * the spectrum lambda (n). */
int coopcg_gen_householder_factors(int n, int m, double kappa, uint64_t seed, double* V,
                                   double* lambda);

/* Host parts of the reference's make_problem<double> (problem.hpp:219-230):
 * the spectrum of random_spd_with_spectrum (problem.hpp:125-139) and
 * random_rhs_and_starts (problem.hpp:187-200: b and X0 uniform on [-10, 10]). */
int coopcg_gen_random_spd_spectrum(int n, double cond, uint64_t seed, double* lambda);
int coopcg_gen_reference_rhs_starts(int n, int p, uint64_t seed, double* b, double* X0_colmajor);

/* Upload b (n) and X0 (n x p column-major) into the context. */
int coopcg_gpu_upload(coopcg_gpu_ctx* ctx, const double* b, const double* X0_colmajor);
/* Run ccg_solve on the resident A, b, X0; fill `trace` (may be NULL). */
int coopcg_gpu_run(coopcg_gpu_ctx* ctx, const coopcg_opts* opts, coopcg_trace* trace);
/* The drop-in: upload + run + copy-out, host buffers in and out. */
int coopcg_gpu_solve(coopcg_gpu_ctx* ctx, const double* b, const double* X0_colmajor,
                     const coopcg_opts* opts, coopcg_trace* trace);

/* ---- verification mode: SolveOptions::keep_history / x_star (trace.hpp:84-87) ----
 * Sticky per context until changed; (0, NULL) turns it off.  Needs one context
 * holding every row of A (not a multi-device handle or a row shard), whole
 * solves (coopcg_gpu_run / _solve), and algo 0 or 2 (not mccg_solve).
 *   keep_history != 0: every solve keeps X_k, R_k, D_k on the device for
 *     k = 0..iterations (entry 0 = the state after setup, entry k + 1 = after
 *     iteration k with D = Dnext: push_history, solvers.hpp:43-50, :146);
 *     3 (max_iters + 1) n P doubles -- the run fails with COOPCG_E_INVALID when
 *     that exceeds half of the free device memory (set max_iters).
 *   x_star != NULL (host, n doubles, copied): every iteration also records
 *     IterationRecord::anorm_errors = ||x_j - x*||_A per agent (block_cg.hpp:316-331,
 *     dense_ops.hpp:159-196) at the cost of one more A.D; exact mode reproduces
 *     the reference's values bit for bit; a quadratic form negative beyond
 *     round-off ends the run with COOPCG_E_SPD_VIOLATION like a_norm's throw. */
int coopcg_gpu_set_verification(coopcg_gpu_ctx* ctx, int keep_history, const double* x_star);
/* History entries of the last run (iterations + 1; 0 without keep_history). */
int coopcg_gpu_history_count(const coopcg_gpu_ctx* ctx, int* entries);
/* Entry `entry` of trace.history_x / _r / _d, each n x p column-major; NULL skips. */
int coopcg_gpu_get_history(coopcg_gpu_ctx* ctx, int entry, double* X_colmajor, double* R_colmajor,
                           double* D_colmajor);
/* Rows 0..min(capacity, iterations) - 1 of the per-iteration A-norm errors, p per row. */
int coopcg_gpu_get_anorm_errors(coopcg_gpu_ctx* ctx, int capacity, double* out);

int coopcg_gpu_timing(const coopcg_gpu_ctx* ctx, coopcg_timing* out);
/* The context's CUDA stream (cudaStream_t), so callers can record events on
 * the stream the kernels run on. */
void* coopcg_gpu_stream(const coopcg_gpu_ctx* ctx);

/* ---- kernel-level entry points (parity tests of the building blocks) ----
 * All take host buffers and run on the context's device/stream. */
/* out = A_rows . D  (D n x p column-major; out (row_end-row_begin) x p column-major) */
int coopcg_gpu_matvec_block(coopcg_gpu_ctx* ctx, const double* D_colmajor, double* out_colmajor);
/* numerical_rank of an n x p column-major block (dense_ops.hpp:104-157). */
int coopcg_gpu_numerical_rank(coopcg_gpu_ctx* ctx, const double* D_colmajor, double tol,
                              int* rank);
/* Same; force_exact != 0 skips the Gram certificate and always runs the
 * exact column-pivoted MGS restatement (tests of both paths). */
int coopcg_gpu_numerical_rank_ex(coopcg_gpu_ctx* ctx, const double* D_colmajor, double tol,
                                 int force_exact, int* rank);

/* ---- row-sharded (multi-GPU) driving -------------------------------------
 * A context created with coopcg_gpu_create_shard owns rows [row_begin,
 * row_end) of A; all n x p blocks are replicated.  The caller runs a solve as
 *   begin; SETUP_LOCAL; <all-gather R rows>; SETUP_REST;
 *   for k: ITER_LOCAL(k); <all-gather Q rows>; ITER_MID(k);
 *          if recompute_at(k): <all-gather R rows>;  ITER_REST(k);
 *          (poll coopcg_gpu_state now and then; after a stop, phases are no-ops)
 *   FINAL_LOCAL; <all-gather S rows>; FINAL_REST; end.
 * mccg_solve (opts.algo = 1) adds MCCG_SETUP right after SETUP_REST, and
 * after a polled stop a call to coopcg_gpu_mccg_resume: when the stop was a
 * rank drop it restricts the agents (solvers.hpp:156-175; every rank holds
 * the same replicated blocks, so every rank restricts identically) and
 * returns the iteration to continue from, else -1. 
 * A "local" phase writes only this context's rows of the named block;
 * coopcg_gpu_block returns the device pointer (row-major, leading dimension
 * `ld` doubles) for the exchange.  All work is ordered on the context stream
 * (coopcg_gpu_stream).  DESIGN.md §7; paper_1204_0069_b200/sharded.py. */
enum coopcg_phase {
    COOPCG_PH_SETUP_LOCAL = 0, COOPCG_PH_SETUP_REST = 1,
    COOPCG_PH_ITER_LOCAL = 2, COOPCG_PH_ITER_MID = 3, COOPCG_PH_ITER_REST = 4,
    COOPCG_PH_FINAL_LOCAL = 5, COOPCG_PH_FINAL_REST = 6,
    COOPCG_PH_MCCG_SETUP = 7  /* mccg: setup_coordinator's restriction (solvers.hpp:63-91) */
};
enum coopcg_block { COOPCG_BLOCK_X = 0, COOPCG_BLOCK_R = 1, COOPCG_BLOCK_D = 2, COOPCG_BLOCK_Q = 3, COOPCG_BLOCK_S = 4,
                    COOPCG_BLOCK_W = 5 /* Householder generation's w vector (n x 1, ld 1) */ };
int coopcg_gpu_begin(coopcg_gpu_ctx* ctx, const coopcg_opts* opts);
int coopcg_gpu_phase(coopcg_gpu_ctx* ctx, int phase, int k);
int coopcg_gpu_recompute_at(const coopcg_gpu_ctx* ctx, int k);
int coopcg_gpu_block(coopcg_gpu_ctx* ctx, int which, int k, void** dev_ptr, int* ld);
int coopcg_gpu_state(coopcg_gpu_ctx* ctx, int* stop, int* iterations);
/* mccg after a polled stop: *next_k = iteration to resume from (the agents
 * were restricted), or -1 (the solve is over). */
int coopcg_gpu_mccg_resume(coopcg_gpu_ctx* ctx, int* next_k);
int coopcg_gpu_end(coopcg_gpu_ctx* ctx, coopcg_trace* trace);

/* ---- peer-memory Q exchange (one process per GPU, NVLink / NVSwitch) ------
 * Replaces the per-iteration all-gather of Q: the kernel that computes this
 * rank's rows of Q (the A.D epilogue, or the fast row pass) stores them into
 * every rank's Q through CUDA IPC mappings, so after a stream-ordered barrier
 * (a tiny NCCL all-reduce, or a host barrier) every rank holds the full Q.
 * In this mode Q is double-buffered by iteration parity (coopcg_gpu_block
 * returns the buffer of iteration k), so no rank overwrites rows a slower rank
 * still reads.  R and S keep their all-gathers (setup, recompute, final).
 *   coopcg_gpu_ipc_handles: this context's two Q buffers as two 64-byte
 *     cudaIpcMemHandle_t (written to handles_out[0..127]).
 *   coopcg_gpu_set_peers: `handles` holds nranks x 128 bytes (rank order);
 *     the context maps every other rank's buffers (own slot ignored) and
 *     switches to peer mode.  nranks <= 8. */
#define COOPCG_IPC_HANDLE_BYTES 64
int coopcg_gpu_ipc_handles(coopcg_gpu_ctx* ctx, void* handles_out);
int coopcg_gpu_set_peers(coopcg_gpu_ctx* ctx, int nranks, int self_rank, const void* handles);

/* ---- multi-GPU inside the library --------------------------
 * A is split into row blocks (coopcg_row_split: even blocks, rounded to 64-row
 * panels); every n x p block and the p x p state are replicated, each shard
 * computes its rows of Q = A_g D and the rows are exchanged once per
 * iteration (plus R at setup / recompute iterations and S at finalize).  The
 * run loop enqueues every shard's work and every exchange from the library:
 * no per-iteration call from the host program.  In exact mode the result is
 * bit-identical to one GPU for any split (each row's A-chain is local).
 *
 * coopcg_gpu_create_multi: ONE process drives ndev devices (a device may
 *   repeat, e.g. two shards on one GPU).  The kernel that computes a shard's
 *   rows of Q stores them into every shard's Q over NVLink / NVSwitch peer
 *   memory (cudaDeviceEnablePeerAccess), so the exchange is a cross-stream
 *   event barrier, not a collective.  The handle takes the whole-matrix calls:
 *   set_A (all n rows), gen_A (DIAGDOM, HOUSEHOLDER), get_A[_rows], upload, run,
 *   solve, timing, matvec_block, numerical_rank; not the phase API.
 * coopcg_gpu_create_rank: ONE process per GPU (e.g. under torchrun); rank
 *   `rank` of `nranks` owns coopcg_row_split's block `rank`, and the row
 *   exchanges are NCCL collectives (grouped in-place broadcasts = an
 *   all-gather of row blocks) on the context stream, enqueued by
 *   coopcg_gpu_run.  Every rank calls create / gen_A or set_A (its own rows) /
 *   upload / run with identical arguments.  `nccl_id` is
 *   COOPCG_NCCL_ID_BYTES bytes from coopcg_nccl_unique_id on one rank,
 *   distributed by the caller.  NCCL is loaded on first use (libnccl.so.2). */
#define COOPCG_NCCL_ID_BYTES 128
int coopcg_row_split(int n, int parts, int part, int* row_begin, int* row_end);
int coopcg_gpu_create_multi(int n, int p, int ndev, const int* devices, int arith, coopcg_gpu_ctx** out);
int coopcg_nccl_unique_id(void* id_out);
int coopcg_gpu_create_rank(int n, int p, int device, int arith, int nranks, int rank, const void* nccl_id,
                           coopcg_gpu_ctx** out);
/* Shards of a context (1 for a single-device or rank context): count, and
 * for the first `cap` shards their device and row block. */
int coopcg_gpu_shards(const coopcg_gpu_ctx* ctx, int cap, int* nshards, int* devices, int* row_begin,
                      int* row_end);

#ifdef __cplusplus
}
#endif
#endif /* COOPCG_GPU_H */
