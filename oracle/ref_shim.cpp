// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/build_ref.sh compiles this file against
// /root/reference/proj/include (header-only library; no reference sources
// are copied into this repo) into oracle/_ref/libccgref.so, which the tests
// use to pin the C restatement (oracle/ccg_oracle.c) and to make the golden
// fixtures, and which bench.py times as the reference CPU baseline.
//
// Entry points mirror the reference API:
//   ccg_solve      coopcg/solvers.hpp:329-333
//   parallel_ccg   coopcg/parallel.hpp:76-111
//   mccg_solve     coopcg/solvers.hpp:338-342
//   cg_solve       coopcg/solvers.hpp:388-530
//   make_problem   coopcg/problem.hpp:234-246
//   matvec_block / gram / solve_small / numerical_rank  coopcg/dense_ops.hpp
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <vector>

#include <sys/mman.h>

#include "coopcg/parallel.hpp"
#include "coopcg/problem.hpp"
#include "coopcg/solvers.hpp"

extern "C" {
#include "ccg_oracle.h"
}

using namespace coopcg;

namespace {

int status_code(TerminalStatus s) {
    switch (s) {
    case TerminalStatus::Converged: return ORC_STATUS_CONVERGED;
    case TerminalStatus::RankCollapse: return ORC_STATUS_RANK_COLLAPSE;
    case TerminalStatus::MaxIterations: return ORC_STATUS_MAX_ITERATIONS;
    }
    return -1;
}

template <class F>
int guarded(orc_trace* tr, F&& f) {
    try {
        f();
        return ORC_OK;
    } catch (const SpdViolationError& e) {
        std::snprintf(tr->error_msg, sizeof tr->error_msg, "%s", e.what());
        return ORC_E_SPD_VIOLATION;
    } catch (const NumericalBreakdownError& e) {
        std::snprintf(tr->error_msg, sizeof tr->error_msg, "%s", e.what());
        return ORC_E_NUMERICAL_BREAKDOWN;
    } catch (const DimensionError& e) {
        std::snprintf(tr->error_msg, sizeof tr->error_msg, "%s", e.what());
        return ORC_E_DIMENSION;
    } catch (const std::exception& e) {
        std::snprintf(tr->error_msg, sizeof tr->error_msg, "%s", e.what());
        return 9;
    }
}

void fill_trace(const SolveTrace<double>& t, int n, orc_trace* tr) {
    tr->status = status_code(t.status);
    tr->converged_agent = t.converged_agent;
    tr->iterations = t.iteration_count();
    tr->loop_wall_ns = t.loop_wall_ns;
    const int p0 = t.initial_residual_norms.empty() ? 0 : (int)t.initial_residual_norms.size();
    for (int k = 0; k < tr->iterations && k < tr->capacity; ++k) {
        const auto& rec = t.iterations[(size_t)k];
        // Norms are stored per ORIGINAL agent id so restricted (mccg) traces
        // keep a fixed p-wide row; inactive agents are NaN.
        if (tr->residual_norms) {
            for (int j = 0; j < p0; ++j) tr->residual_norms[(size_t)k * p0 + j] = __builtin_nan("");
            for (int s = 0; s < rec.active_agents; ++s)
                tr->residual_norms[(size_t)k * p0 + rec.agents[(size_t)s]] = rec.residual_norms[(size_t)s];
        }
        if (tr->minres) tr->minres[k] = rec.minres;
        if (tr->wall_ns) tr->wall_ns[k] = rec.wall_ns;
    }
    if (tr->initial_residual_norms)
        std::copy(t.initial_residual_norms.begin(), t.initial_residual_norms.end(), tr->initial_residual_norms);
    tr->initial_minres = t.initial_minres;
    if (tr->final_x) {
        // final_x is n x (surviving agents), column-major; scatter by agent id
        // (NaN columns for agents a restriction dropped).
        for (size_t e = 0; e < static_cast<size_t>(n) * p0; ++e) tr->final_x[e] = __builtin_nan("");
        for (int s = 0; s < t.final_x.cols(); ++s) {
            auto c = t.final_x.col(s);
            std::copy(c.begin(), c.end(), tr->final_x + (size_t)t.active_agents[(size_t)s] * n);
        }
    }
    if (tr->active_agents)
        for (size_t s = 0; s < t.active_agents.size(); ++s) tr->active_agents[s] = t.active_agents[s];
    tr->n_active = static_cast<int>(t.active_agents.size());
    if (tr->final_residual_norms) {
        for (int j = 0; j < p0; ++j) tr->final_residual_norms[j] = __builtin_nan("");
        for (size_t s = 0; s < t.final_residual_norms.size(); ++s)
            tr->final_residual_norms[t.active_agents[s]] = t.final_residual_norms[s];
    }
    tr->final_minres = t.final_minres;
}

SpdMatrix<double> make_A(int n, const double* A) {
    return SpdMatrix<double>(n, std::vector<double>(A, A + (size_t)n * n), SpdCheck::skip);
}

// A system matrix owned by the shim, for the full-size BASELINE configs
// (A = 34 / 137 GB at cfg 3 / 4): the caller fills the entries in place
// (ref_matrix_data) and the vector is then MOVED into the reference's
// SpdMatrix (SpdCheck::skip: the generators are exactly symmetric, so the
// float-mode symmetrisation would be the identity, dense.hpp:104-122), so
// the host holds one copy of A, not two as make_A does.
struct RefMatrix {
    int n = 0;
    double* data = nullptr;
    std::vector<double> v;
    std::optional<SpdMatrix<double>> m;
    const SpdMatrix<double>& sealed() {
        if (!m) {
            m.emplace(n, std::move(v), SpdCheck::skip);
            data = const_cast<double*>(m->entries().data());
        }
        return *m;
    }
};

// parallel_ccg (parallel.hpp:76-111) with one change, for the full-size
// BASELINE configs only: finalize_trace's per-agent loop (solvers.hpp:188-210:
// A x_j - b and its 2-norm, one agent after another in the coordinator) is run
// by the team, agent j on worker j, with the reference's own kernels::matvec_col
// and kernels::norm2.  Each agent's residual is the same sequence of operations
// either way, so the trace is bit-identical to parallel_ccg's (pinned by
// tests/test_oracle.py::test_team_finalize_equals_parallel_ccg); at cfg 4 the
// serial loop is 32 latency-bound 131072^2 matvecs (~9 minutes), the team's ~1.
// Every other step is the reference's: its drive() loop and OmpExecutor, wrapped.
template <ScalarField S>
class TeamFinalizeExecutor {
public:
    TeamFinalizeExecutor(detail::BlockCgWorkspace<S>& ws, detail::DriverControl& ctrl, SolveTrace<S>& trace,
                         std::vector<double>& fres, int tid)
        : inner_(ws, ctrl, tid), ws_(&ws), ctrl_(&ctrl), trace_(&trace), fres_(&fres), tid_(tid) {}
    template <class F>
    void phase(F&& f) { inner_.phase(std::forward<F>(f)); }
    void barrier() { inner_.barrier(); }
    template <class F>
    void coordinator(F&& f) {
        // drive() enters a coordinator section with ctrl.stop already set only
        // for finalize_trace (every other one sets it, solvers.hpp:264-283)
        if (!ctrl_->stop) {
            inner_.coordinator(std::forward<F>(f));
            return;
        }
        inner_.barrier();
        const bool failed = ctrl_->worker_failed.load(std::memory_order_seq_cst);
        if (!failed && tid_ < ws_->p) {
            const int j = tid_;
            Vec<S> scratch(static_cast<std::size_t>(ws_->n));
            kernels::matvec_col<S>(*ws_->A, ws_->X.col(j), std::span<S>(scratch.data(), scratch.size()));
            for (int i = 0; i < ws_->n; ++i)
                scratch[static_cast<std::size_t>(i)] -= (*ws_->b)[static_cast<std::size_t>(i)];
            (*fres_)[static_cast<std::size_t>(j)] =
                kernels::norm2<S>(std::span<const S>(scratch.data(), scratch.size()));
        }
        inner_.barrier();
#pragma omp single
        {
            trace_->status = ctrl_->status;
            trace_->converged_agent = ctrl_->converged_agent;
            trace_->final_x = ws_->X;
            trace_->active_agents = ws_->agent_ids;
            if (!failed) {
                trace_->final_residual_norms.assign(fres_->begin(), fres_->begin() + ws_->p);
                trace_->final_minres = trace_->final_residual_norms.empty()
                                           ? 0.0
                                           : *std::min_element(trace_->final_residual_norms.begin(),
                                                               trace_->final_residual_norms.end());
            }
        }
    }

private:
    detail::OmpExecutor<S> inner_;
    detail::BlockCgWorkspace<S>* ws_;
    detail::DriverControl* ctrl_;
    SolveTrace<S>* trace_;
    std::vector<double>* fres_;
    int tid_;
};

SolveTrace<double> parallel_ccg_team_finalize(const SpdMatrix<double>& A, const Vec<double>& b,
                                              const DenseBlock<double>& X0, const SolveOptions<double>& opts) {
    // the body of parallel_ccg (parallel.hpp:79-110) with the wrapped executor
    detail::check_block_inputs(A, b, X0);
    const int p = X0.cols();
    detail::BlockCgWorkspace<double> ws;
    ws.init(A, b, X0);
    detail::DriverControl ctrl;
    ctrl.max_iters = detail::resolve_max_iters(opts, A.dim());
    SolveTrace<double> trace;
    const int recompute_every = detail::resolve_recompute(opts, 50);
    std::vector<double> fres(static_cast<std::size_t>(p));
    bool team_ok = true;
    omp_set_dynamic(0);
#pragma omp parallel num_threads(p) default(shared)
    {
        if (omp_get_num_threads() != p) {
#pragma omp single
            team_ok = false;
        } else {
            TeamFinalizeExecutor<double> exec(ws, ctrl, trace, fres, omp_get_thread_num());
            detail::drive(ws, ctrl, trace, opts, recompute_every, /*allow_restriction=*/false, exec);
        }
    }
    if (!team_ok) throw Error("parallel_ccg: could not start " + std::to_string(p) + " workers");
    detail::rethrow_pending(ctrl);
    trace.barriers_per_iteration = WorkPlan::standard(p).barriers_per_iteration();
    return trace;
}

int block_solve(int algo, const SpdMatrix<double>& Am, int n, int p, const double* b, const double* X0,
                const orc_opts* o, orc_trace* tr) {
    std::vector<double> bv(b, b + n);
    DenseBlock<double> x0(n, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i) x0(i, j) = X0[(size_t)j * n + i];
    SolveOptions<double> opts;
    opts.tol = o->tol;
    opts.max_iters = o->max_iters;
    opts.recompute_residual_every = o->recompute_residual_every;
    opts.rank_rel_tol = o->rank_rel_tol;
    SolveTrace<double> t;
    if (algo == 0) t = ccg_solve(Am, bv, x0, opts);
    else if (algo == 1) t = parallel_ccg(Am, bv, x0, opts, p);
    else if (algo == 3) t = parallel_ccg_team_finalize(Am, bv, x0, opts);
    else t = mccg_solve(Am, bv, x0, opts);
    fill_trace(t, n, tr);
    return 0;
}

} // namespace

extern "C" {

/// A shim-owned n x n matrix (row-major entries, filled by the caller through
/// ref_matrix_data before the first solve).  NULL if the allocation fails.
void* ref_matrix_new(int n) {
    try {
        auto* h = new RefMatrix;
        h->n = n;
        const size_t N = static_cast<size_t>(n) * n;
        // reserve (mmap, untouched), ask for transparent huge pages and fault
        // the pages in from every core: resize()'s single-threaded zero fill
        // of up to 137 GB then runs on mapped memory instead of taking 4 KB
        // page faults one at a time
        h->v.reserve(N);
        {
            const uintptr_t a = reinterpret_cast<uintptr_t>(h->v.data());
            const uintptr_t lo = (a + 4095) & ~uintptr_t(4095), hi = (a + N * sizeof(double)) & ~uintptr_t(4095);
            if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
            char* base = reinterpret_cast<char*>(h->v.data());
            const size_t bytes = N * sizeof(double), chunk = size_t(64) << 20;
#pragma omp parallel for schedule(dynamic, 1)
            for (long long c = 0; c < (long long)((bytes + chunk - 1) / chunk); ++c) {
                const size_t o = (size_t)c * chunk;
                std::memset(base + o, 0, std::min(chunk, bytes - o));
            }
        }
        h->v.resize(N);
        h->data = h->v.data();
        return h;
    } catch (...) {
        return nullptr;
    }
}

double* ref_matrix_data(void* h) { return static_cast<RefMatrix*>(h)->data; }

void ref_matrix_free(void* h) { delete static_cast<RefMatrix*>(h); }

/// ref_block_solve on a shim-owned matrix (no copy of A).
int ref_block_solve_m(int algo, void* h, int p, const double* b, const double* X0, const orc_opts* o,
                      orc_trace* tr) {
    tr->error_msg[0] = '\0';
    auto* rm = static_cast<RefMatrix*>(h);
    return guarded(tr, [&] { block_solve(algo, rm->sealed(), rm->n, p, b, X0, o, tr); });
}

/// algo: 0 = ccg_solve, 1 = parallel_ccg (p OpenMP threads), 2 = mccg_solve,
/// 3 = parallel_ccg with finalize_trace's agent loop run by the team (above).
int ref_block_solve(int algo, int n, int p, const double* A, const double* b, const double* X0,
                    const orc_opts* o, orc_trace* tr) {
    tr->error_msg[0] = '\0';
    return guarded(tr, [&] { block_solve(algo, make_A(n, A), n, p, b, X0, o, tr); });
}

int ref_cg_solve(int n, const double* A, const double* b, const double* x0, const orc_opts* o,
                 orc_trace* tr) {
    tr->error_msg[0] = '\0';
    return guarded(tr, [&] {
        auto Am = make_A(n, A);
        std::vector<double> bv(b, b + n), xv(x0, x0 + n);
        SolveOptions<double> opts;
        opts.tol = o->tol;
        opts.max_iters = o->max_iters;
        opts.recompute_residual_every = o->recompute_residual_every;
        opts.rank_rel_tol = o->rank_rel_tol;
        auto t = cg_solve(Am, bv, xv, opts);
        fill_trace(t, n, tr);
    });
}

int ref_sd_solve(int n, const double* A, const double* b, const double* x0, const orc_opts* o,
                 orc_trace* tr) {
    tr->error_msg[0] = '\0';
    return guarded(tr, [&] {
        auto Am = make_A(n, A);
        std::vector<double> bv(b, b + n), xv(x0, x0 + n);
        SolveOptions<double> opts;
        opts.tol = o->tol;
        opts.max_iters = o->max_iters;
        opts.recompute_residual_every = o->recompute_residual_every;
        auto t = steepest_descent_solve(Am, bv, xv, opts);
        fill_trace(t, n, tr);
    });
}

/// The reference's own problem family (random_spd + rhs/starts, float mode).
int ref_make_problem(int n, int p, double cond, unsigned long long seed, double* A, double* b,
                     double* X0) {
    try {
        ProblemSpec spec;
        spec.n = n;
        spec.p = p;
        spec.cond = cond;
        spec.seed = seed;
        auto inst = make_problem<double>(spec);
        std::copy(inst.A.entries().begin(), inst.A.entries().end(), A);
        std::copy(inst.b.begin(), inst.b.end(), b);
        for (int j = 0; j < p; ++j) {
            auto c = inst.X0.col(j);
            std::copy(c.begin(), c.end(), X0 + (size_t)j * n);
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

// random_spd_with_spectrum(n, cond, seed) (problem.hpp:118-152): A and the spectrum.
int ref_random_spd(int n, double cond, unsigned long long seed, double* A, double* lambda) {
    try {
        auto gen = random_spd_with_spectrum(n, cond, seed);
        std::copy(gen.A.entries().begin(), gen.A.entries().end(), A);
        std::copy(gen.spectrum.begin(), gen.spectrum.end(), lambda);
        return 0;
    } catch (...) {
        return 1;
    }
}

void ref_matvec_block(int n, int p, const double* A, const double* D, double* out) {
    auto Am = make_A(n, A);
    DenseBlock<double> d(n, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i) d(i, j) = D[(size_t)j * n + i];
    auto q = matvec_block(Am, d);
    for (int j = 0; j < p; ++j) {
        auto c = q.col(j);
        std::copy(c.begin(), c.end(), out + (size_t)j * n);
    }
}

void ref_gram(int n, int p, const double* D, const double* AD, double* raw, double* sym) {
    DenseBlock<double> d(n, p), ad(n, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i) {
            d(i, j) = D[(size_t)j * n + i];
            ad(i, j) = AD[(size_t)j * n + i];
        }
    auto r = gram_raw(d, ad);
    auto s = gram(d, ad);
    std::copy(r.data().begin(), r.data().end(), raw);
    std::copy(s.data().begin(), s.data().end(), sym);
}

/// Returns 0 on success, 1 on SingularMatrixError.
int ref_solve_small(int p, const double* M, int q, const double* B, double* X) {
    SmallSpd<double> m(p);
    std::copy(M, M + (size_t)p * p, m.data().begin());
    DenseBlock<double> bb(p, q);
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) bb(i, j) = B[(size_t)j * p + i];
    try {
        auto x = solve_small(m, bb);
        for (int j = 0; j < q; ++j)
            for (int i = 0; i < p; ++i) X[(size_t)j * p + i] = x(i, j);
        return 0;
    } catch (const SingularMatrixError&) {
        return 1;
    }
}

int ref_numerical_rank(int n, int p, const double* D, double tol, int* columns) {
    DenseBlock<double> d(n, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i) d(i, j) = D[(size_t)j * n + i];
    auto r = numerical_rank(d, tol);
    if (columns)
        std::copy(r.columns.begin(), r.columns.end(), columns);
    return r.rank;
}

} // extern "C"
