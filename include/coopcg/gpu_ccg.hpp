// gpu_ccg.hpp -- C++ drop-in for the reference's ccg_solve on a B200.
//
// Header-only wrapper over the C ABI (coopcg_gpu.h).  It includes the
// reference's own headers (coopcg/solvers.hpp and what it pulls in) and
// returns the reference's SolveTrace<double>, so a caller switches with
//
//     auto t = coopcg::ccg_solve(A, b, X0, opts);          // CPU reference
//     auto t = coopcg::gpu_ccg(A, b, X0, opts);            // this library
//
// Semantics follow ccg_solve (coopcg/solvers.hpp:325-333): the same shape
// checks and DimensionError messages (solvers.hpp:300-306), the same statuses
// (trace.hpp:13-17), SpdViolationError for a nonpositive direction energy
// (solvers.hpp:111-115), per-iteration records with the reference's mult
// counting (workplan.hpp:693-715), final_residual_norms by true
// recomputation (solvers.hpp:188-210).  In the default exact arithmetic mode
// the trace is bit-identical to ccg_solve's, including the
// verification mode (trace.hpp:84-87): keep_history fills history_x / _r / _d
// and x_star the per-iteration anorm_errors (one device, not gpu_mccg, which
// rejects them with std::invalid_argument rather than ignoring them).
//
// GpuSolver keeps A resident on the device between solves (SpdMatrix is
// immutable, dense.hpp:95-96), the common "many right-hand sides" use.
// gpu_make_problem is make_problem<double> with the matrix generated on the
// device (the reference's Haar-MGS random_spd is O(n^3) and serial on a CPU).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "coopcg/problem.hpp"
#include "coopcg/solvers.hpp"
#include "coopcg_gpu.h"

namespace coopcg {

struct GpuOptions {
    enum class Arith { exact, fast };
    int device = 0;
    Arith arith = Arith::exact;
    /// More than one entry: A is row-block sharded over these devices, all
    /// driven by this process (coopcg_gpu_create_multi; the A.D kernel stores
    /// its Q rows into every device's Q over NVLink).  Empty: `device` alone.
    std::vector<int> devices;
};

namespace gpu_detail {

[[noreturn]] inline void raise(int rc, const std::string& msg) {
    switch (rc) {
    case COOPCG_E_DIMENSION: throw DimensionError(msg);
    case COOPCG_E_SPD_VIOLATION: throw SpdViolationError(msg);
    case COOPCG_E_NUMERICAL_BREAKDOWN: throw NumericalBreakdownError(msg);
    case COOPCG_E_SINGULAR: throw SingularMatrixError(msg);
    default: throw Error("coopcg_gpu: " + msg);
    }
}

inline std::string last_error(const coopcg_gpu_ctx* ctx) {
    char buf[512];
    coopcg_gpu_last_error(ctx, buf, sizeof buf);
    return buf;
}

inline TerminalStatus status_of(int s) {
    switch (s) {
    case COOPCG_CONVERGED: return TerminalStatus::Converged;
    case COOPCG_RANK_COLLAPSE: return TerminalStatus::RankCollapse;
    default: return TerminalStatus::MaxIterations;
    }
}

}  // namespace gpu_detail

/// A context bound to one matrix on one GPU; solve() may be called repeatedly.
class GpuSolver {
public:
    GpuSolver(const SpdMatrix<double>& A, int p, const GpuOptions& g = {}) : n_(A.dim()), p_(p) {
        const int arith = g.arith == GpuOptions::Arith::fast ? COOPCG_ARITH_FAST : COOPCG_ARITH_EXACT;
        if (p < 1 || p >= n_) throw DimensionError("solver: need 1 <= p < n starting columns");
        int rc = g.devices.size() > 1
                     ? coopcg_gpu_create_multi(n_, p, static_cast<int>(g.devices.size()), g.devices.data(), arith, &ctx_)
                     : coopcg_gpu_create(n_, p, g.devices.empty() ? g.device : g.devices[0], arith, &ctx_);
        if (rc != COOPCG_OK) gpu_detail::raise(rc, gpu_detail::last_error(nullptr));
        rc = coopcg_gpu_set_A(ctx_, A.entries().data());
        if (rc != COOPCG_OK) {
            const std::string m = gpu_detail::last_error(ctx_);
            coopcg_gpu_destroy(ctx_);
            gpu_detail::raise(rc, m);
        }
    }
    GpuSolver(const GpuSolver&) = delete;
    GpuSolver& operator=(const GpuSolver&) = delete;
    ~GpuSolver() { coopcg_gpu_destroy(ctx_); }

    /// algo 0: ccg_solve semantics; 1: mccg_solve (restriction on rank drop).
    SolveTrace<double> solve(const Vec<double>& b, const DenseBlock<double>& X0, const SolveOptions<double>& opts = {},
                             int algo = 0) {
        // check_block_inputs (solvers.hpp:300-306)
        if (static_cast<int>(b.size()) != n_ || X0.rows() != n_)
            throw DimensionError("solver: operand shapes do not match the system matrix");
        if (X0.cols() < 1 || X0.cols() >= n_) throw DimensionError("solver: need 1 <= p < n starting columns");
        if (X0.cols() != p_) throw DimensionError("gpu_ccg: agent count differs from the solver's");
        // Verification mode (trace.hpp:84-87: history blocks, A-norm errors against
        // an oracle solution): coopcg_gpu_set_verification; one device, not mccg.
        const bool verify = opts.keep_history || opts.x_star != nullptr;
        if (verify && algo == 1)
            throw std::invalid_argument("gpu_mccg: keep_history / x_star (verification mode) are not supported "
                                        "on the GPU backend; use mccg_solve for invariant checks");
        if (opts.x_star != nullptr && static_cast<int>(opts.x_star->size()) != n_)
            throw DimensionError("solver: operand shapes do not match the system matrix");
        if (verify || verify_on_) {
            const int vrc = coopcg_gpu_set_verification(ctx_, opts.keep_history ? 1 : 0,
                                                        opts.x_star ? opts.x_star->data() : nullptr);
            if (vrc != COOPCG_OK) gpu_detail::raise(vrc, gpu_detail::last_error(ctx_));
            verify_on_ = verify;
        }
        const int n = n_, p = p_;
        const int max_iters = opts.max_iters >= 0 ? opts.max_iters : 2 * n;  // solvers.hpp:18-23
        const int cap = max_iters > 0 ? max_iters : 1;
        std::vector<double> norms(static_cast<size_t>(cap) * p), minres(cap), init(p), fres(p);
        std::vector<uint64_t> wall(cap);
        // DenseBlock is one contiguous column-major buffer (dense.hpp:105-155).
        std::vector<double> x0(static_cast<size_t>(n) * p), fx(static_cast<size_t>(n) * p);
        for (int j = 0; j < p; ++j) {
            auto c = X0.col(j);
            std::copy(c.begin(), c.end(), x0.begin() + static_cast<size_t>(j) * n);
        }
        coopcg_opts o{opts.tol, opts.max_iters, opts.recompute_residual_every, opts.rank_rel_tol, algo};
        std::vector<int> act(p);
        coopcg_trace tr{};
        tr.active_agents = act.data();
        tr.capacity = cap;
        tr.residual_norms = norms.data();
        tr.minres = minres.data();
        tr.wall_ns = wall.data();
        tr.initial_residual_norms = init.data();
        tr.final_x = fx.data();
        tr.final_residual_norms = fres.data();
        const int rc = coopcg_gpu_solve(ctx_, b.data(), x0.data(), &o, &tr);
        if (rc != COOPCG_OK) gpu_detail::raise(rc, gpu_detail::last_error(ctx_));

        SolveTrace<double> t;
        const int every = opts.recompute_residual_every >= 0 ? opts.recompute_residual_every : 50;
        for (int k = 0; k < tr.iterations; ++k) {
            // rows hold norms per ORIGINAL agent id, NaN for agents mccg dropped
            IterationRecord rec;
            rec.k = k;
            for (int j = 0; j < p; ++j) {
                const double v = norms[static_cast<size_t>(k) * p + j];
                if (!std::isnan(v)) {
                    rec.agents.push_back(j);
                    rec.residual_norms.push_back(v);
                }
            }
            rec.active_agents = static_cast<int>(rec.agents.size());
            rec.minres = minres[k];
            const bool rcmp = detail::recompute_now(k, every);
            std::uint64_t m = 0;
            for (int ph = 0; ph < kPhaseCount; ++ph)
                m += phase_counted_mults(static_cast<Phase>(ph), n, rec.active_agents, rcmp);
            rec.mults = m;
            rec.mults_per_worker.assign(rec.active_agents, m);
            rec.wall_ns = wall[k];
            t.iterations.push_back(std::move(rec));
        }
        if (opts.x_star != nullptr && tr.iterations > 0) {  // IterationRecord::anorm_errors (solvers.hpp:131)
            std::vector<double> an(static_cast<size_t>(tr.iterations) * p);
            const int arc = coopcg_gpu_get_anorm_errors(ctx_, tr.iterations, an.data());
            if (arc != COOPCG_OK) gpu_detail::raise(arc, gpu_detail::last_error(ctx_));
            for (int k = 0; k < tr.iterations; ++k)
                t.iterations[static_cast<size_t>(k)].anorm_errors.assign(an.begin() + static_cast<size_t>(k) * p,
                                                                         an.begin() + static_cast<size_t>(k + 1) * p);
        }
        if (opts.keep_history) {  // push_history (solvers.hpp:43-50): entry 0 = setup, k + 1 = after iteration k
            int entries = 0;
            coopcg_gpu_history_count(ctx_, &entries);
            std::vector<double> hx(static_cast<size_t>(n) * p), hr(hx.size()), hd(hx.size());
            auto block_of = [&](const std::vector<double>& v) {
                DenseBlock<double> blk(n, p);
                for (int j = 0; j < p; ++j)
                    for (int i = 0; i < n; ++i) blk(i, j) = v[static_cast<size_t>(j) * n + i];
                return blk;
            };
            for (int e = 0; e < entries; ++e) {
                const int hrc = coopcg_gpu_get_history(ctx_, e, hx.data(), hr.data(), hd.data());
                if (hrc != COOPCG_OK) gpu_detail::raise(hrc, gpu_detail::last_error(ctx_));
                t.history_x.push_back(block_of(hx));
                t.history_r.push_back(block_of(hr));
                t.history_d.push_back(block_of(hd));
            }
        }
        t.status = gpu_detail::status_of(tr.status);
        t.converged_agent = tr.converged_agent;
        const int na = tr.n_active;
        t.active_agents.assign(act.begin(), act.begin() + na);
        t.final_x = DenseBlock<double>(n, na);
        for (int s = 0; s < na; ++s)
            for (int i = 0; i < n; ++i) t.final_x(i, s) = fx[static_cast<size_t>(t.active_agents[s]) * n + i];
        t.initial_residual_norms = init;
        t.initial_minres = tr.initial_minres;
        for (int s = 0; s < na; ++s) t.final_residual_norms.push_back(fres[t.active_agents[s]]);
        t.final_minres = tr.final_minres;
        t.setup_mults = static_cast<std::uint64_t>(n) * static_cast<std::uint64_t>(n);
        t.loop_wall_ns = tr.loop_wall_ns;
        t.barriers_per_iteration = 0;
        return t;
    }

private:
    int n_, p_;
    coopcg_gpu_ctx* ctx_ = nullptr;
    bool verify_on_ = false;
};

/// mccg_solve's signature plus GPU options (solvers.hpp:338-342).
inline SolveTrace<double> gpu_mccg(const SpdMatrix<double>& A, const Vec<double>& b, const DenseBlock<double>& X0,
                                   const SolveOptions<double>& opts = {}, const GpuOptions& g = {}) {
    detail::check_block_inputs(A, b, X0);
    GpuSolver s(A, X0.cols(), g);
    return s.solve(b, X0, opts, 1);
}

/// ccg_solve's signature plus GPU options (solvers.hpp:329-333).
inline SolveTrace<double> gpu_ccg(const SpdMatrix<double>& A, const Vec<double>& b, const DenseBlock<double>& X0,
                                  const SolveOptions<double>& opts = {}, const GpuOptions& g = {}) {
    detail::check_block_inputs(A, b, X0);
    GpuSolver s(A, X0.cols(), g);
    return s.solve(b, X0, opts);
}

namespace gpu_detail {

// The scalar solvers on the p = 1 block kernels (algo 0: CG, 2: steepest
// descent), with their own error text and per-iteration mult counting.
inline SolveTrace<double> scalar_solve(const char* name, int algo, const SpdMatrix<double>& A, const Vec<double>& b,
                                       const Vec<double>& x0, SolveOptions<double> opts, const GpuOptions& g) {
    const int n = A.dim();
    if (static_cast<int>(b.size()) != n || static_cast<int>(x0.size()) != n)
        throw DimensionError(std::string(name) + ": operand shapes do not match");
    if (opts.recompute_residual_every < 0) opts.recompute_residual_every = 1;  // solvers.hpp:399, :543
    GpuOptions ge = g;
    if (algo == 2) ge.arith = GpuOptions::Arith::exact;
    SolveTrace<double> t;
    try {
        GpuSolver s(A, 1, ge);
        t = s.solve(b, DenseBlock<double>::from_column(x0), opts, algo);
    } catch (const SpdViolationError& ex) {  // "... at iteration k" from the block path
        const std::string m = ex.what();
        const std::string k = m.substr(m.find_last_of(' ') + 1);
        throw SpdViolationError(std::string(name) + (algo == 2 ? ": nonpositive gradient energy at iteration "
                                                               : ": nonpositive direction energy at iteration ") + k);
    }
    const auto un = static_cast<std::uint64_t>(n);
    for (auto& rec : t.iterations) {  // solvers.hpp:438-486 (CG), :571-603 (SD)
        const bool rc = detail::recompute_now(rec.k, opts.recompute_residual_every);
        const std::uint64_t m = algo == 2 ? (rc ? 2 * un * un + 3 * un + 1 : un * un + 4 * un + 1)
                                          : (rc ? 2 * un * un + 5 * un + 2 : un * un + 6 * un + 2);
        rec.mults = m;
        rec.mults_per_worker.assign(1, m);
    }
    return t;
}

}  // namespace gpu_detail

/// cg_solve's signature plus GPU options (solvers.hpp:388-530): the p = 1 block
/// solver with CG's residual policy reproduces it bit for bit
/// (tests/test_solvers.cpp:176-201 in the reference).
inline SolveTrace<double> gpu_cg_solve(const SpdMatrix<double>& A, const Vec<double>& b, const Vec<double>& x0,
                                       const SolveOptions<double>& opts = {}, const GpuOptions& g = {}) {
    return gpu_detail::scalar_solve("cg_solve", 0, A, b, x0, opts, g);
}

/// steepest_descent_solve's signature plus GPU options (solvers.hpp:532-646);
/// exact arithmetic only.
inline SolveTrace<double> gpu_steepest_descent_solve(const SpdMatrix<double>& A, const Vec<double>& b,
                                                     const Vec<double>& x0, const SolveOptions<double>& opts = {},
                                                     const GpuOptions& g = {}) {
    return gpu_detail::scalar_solve("steepest_descent_solve", 2, A, b, x0, opts, g);
}

/// make_problem<double> (problem.hpp:219-230) with A = random_spd(n, cond, seed)
/// generated on the device, bit-identical to the reference's:
/// the reference's own ProblemInstance, so a benchmark harness switches with
///     auto inst = coopcg::make_problem<double>(spec);      // CPU: O(n^3) serial MGS
///     auto inst = coopcg::gpu_make_problem(spec);           // this library
inline ProblemInstance<double> gpu_make_problem(const ProblemSpec& spec, bool with_oracle = false,
                                                const GpuOptions& g = {}) {
    spec.validate();
    if (spec.n < 2) return make_problem<double>(spec, with_oracle);  // the 1 x 1 case: nothing to generate
    const int n = spec.n, p = spec.p;
    coopcg_gpu_ctx* ctx = nullptr;
    int rc = coopcg_gpu_create(n, 1, g.device, COOPCG_ARITH_EXACT, &ctx);
    if (rc != COOPCG_OK) gpu_detail::raise(rc, gpu_detail::last_error(nullptr));
    std::vector<double> a(static_cast<size_t>(n) * n);
    rc = coopcg_gpu_gen_A(ctx, COOPCG_MATRIX_RANDOM_SPD, spec.seed, 0, spec.cond);
    if (rc == COOPCG_OK) rc = coopcg_gpu_get_A(ctx, a.data());
    if (rc != COOPCG_OK) {
        const std::string msg = gpu_detail::last_error(ctx);
        coopcg_gpu_destroy(ctx);
        gpu_detail::raise(rc, msg);
    }
    coopcg_gpu_destroy(ctx);
    std::vector<double> lam(n), bh(n), x0(static_cast<size_t>(n) * p);
    coopcg_gen_random_spd_spectrum(n, spec.cond, spec.seed, lam.data());
    coopcg_gen_reference_rhs_starts(n, p, spec.seed, bh.data(), x0.data());
    Vec<double> b(bh.begin(), bh.end());
    DenseBlock<double> X0(n, p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < n; ++i) X0(i, j) = x0[static_cast<size_t>(j) * n + i];
    const auto [lo, hi] = std::minmax_element(lam.begin(), lam.end());
    // SpdMatrix's float-mode construction symmetrises (already exact) and probes, as random_spd's does
    ProblemInstance<double> inst{SpdMatrix<double>(n, std::move(a)), std::move(b), std::move(X0), std::nullopt,
                                 *hi / *lo};
    if (with_oracle)
        inst.x_star = solve_dense(inst.A, inst.b);
    return inst;
}

}  // namespace coopcg
