// dropin_test.cpp -- TEST INFRASTRUCTURE.  Compares the C++ drop-in
// coopcg::gpu_ccg (include/coopcg/gpu_ccg.hpp) with the reference's own
// coopcg::ccg_solve, field by field, bit for bit (exact mode), through the
// reference's types.  Built by `make -C oracle dropin` against the reference
// headers (this container); the binary travels to the GPU box and
// tests/test_gpu_dropin.py runs it.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "coopcg/gpu_ccg.hpp"
#include "coopcg/problem.hpp"
#include "coopcg/solvers.hpp"

using namespace coopcg;

static int failures = 0;

static bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

static void compare(const char* name, const SolveTrace<double>& r, const SolveTrace<double>& g) {
    bool ok = r.status == g.status && r.converged_agent == g.converged_agent &&
              r.iteration_count() == g.iteration_count() && r.final_x == g.final_x &&
              r.active_agents == g.active_agents && r.setup_mults == g.setup_mults &&
              same(r.initial_minres, g.initial_minres) && same(r.final_minres, g.final_minres) &&
              r.initial_residual_norms.size() == g.initial_residual_norms.size() &&
              r.final_residual_norms.size() == g.final_residual_norms.size();
    for (size_t i = 0; ok && i < r.initial_residual_norms.size(); ++i)
        ok = same(r.initial_residual_norms[i], g.initial_residual_norms[i]);
    for (size_t i = 0; ok && i < r.final_residual_norms.size(); ++i)
        ok = same(r.final_residual_norms[i], g.final_residual_norms[i]);
    for (int k = 0; ok && k < r.iteration_count(); ++k) {
        const auto& a = r.iterations[k];
        const auto& b = g.iterations[k];
        ok = a.k == b.k && a.active_agents == b.active_agents && a.agents == b.agents && same(a.minres, b.minres) &&
             a.mults == b.mults && a.mults_per_worker == b.mults_per_worker &&
             a.residual_norms.size() == b.residual_norms.size();
        for (size_t j = 0; ok && j < a.residual_norms.size(); ++j) ok = same(a.residual_norms[j], b.residual_norms[j]);
    }
    std::printf("%-34s %-14s it=%4d  %s\n", name, to_string(g.status), g.iteration_count(), ok ? "bit-identical" : "MISMATCH");
    if (!ok) ++failures;
}

int main() {
    struct Case { int n, p; double cond; unsigned long long seed; double tol; int max_iters; int recompute; };
    const Case cases[] = {
        {60, 3, 1e2, 1, 1e-8, -1, -1}, {120, 4, 1e3, 7, 1e-9, -1, -1}, {150, 8, 1e4, 3, 1e-8, -1, -1},
        {200, 1, 1e3, 5, 1e-10, -1, -1}, {96, 4, 1e3, 7, 1e-8, -1, 1}, {96, 4, 1e3, 7, 1e-8, -1, 0},
        {300, 16, 1e2, 11, 0.0, 40, -1}, {128, 32, 1e1, 12, 1e-12, -1, -1},
    };
    for (const auto& c : cases) {
        ProblemSpec spec;
        spec.n = c.n;
        spec.p = c.p;
        spec.cond = c.cond;
        spec.seed = c.seed;
        auto inst = make_problem<double>(spec);
        SolveOptions<double> o;
        o.tol = c.tol;
        o.max_iters = c.max_iters;
        o.recompute_residual_every = c.recompute;
        char name[96];
        std::snprintf(name, sizeof name, "make_problem n=%d p=%d cond=%.0e", c.n, c.p, c.cond);
        compare(name, ccg_solve(inst.A, inst.b, inst.X0, o), gpu_ccg(inst.A, inst.b, inst.X0, o));
    }
    {   // degenerate start: x0 = 0 for every agent -> rank collapse at k = 0
        ProblemSpec spec;
        spec.n = 80;
        spec.p = 3;
        spec.cond = 10.0;
        spec.seed = 2;
        auto inst = make_problem<double>(spec);
        DenseBlock<double> z(80, 3);
        SolveOptions<double> o;
        o.tol = 1e-8;
        compare("degenerate x0 = 0", ccg_solve(inst.A, inst.b, z, o), gpu_ccg(inst.A, inst.b, z, o));
        // A row-block sharded over two (here: the same) devices from this process
        GpuOptions g2;
        g2.devices = {0, 0};
        SolveOptions<double> o2;
        o2.tol = 1e-10;
        compare("gpu_ccg devices={0,0}", ccg_solve(inst.A, inst.b, inst.X0, o2), gpu_ccg(inst.A, inst.b, inst.X0, o2, g2));
        GpuOptions g3;
        g3.devices = {0, 0, 0};
        compare("gpu_mccg devices={0,0,0}", mccg_solve(inst.A, inst.b, inst.X0, o2),
                gpu_mccg(inst.A, inst.b, inst.X0, o2, g3));
        // GpuSolver: A resident, two right-hand sides
        GpuSolver s(inst.A, 3);
        compare("GpuSolver reuse #1", ccg_solve(inst.A, inst.b, inst.X0, o), s.solve(inst.b, inst.X0, o));
        compare("GpuSolver reuse #2", ccg_solve(inst.A, inst.b, inst.X0, o), s.solve(inst.b, inst.X0, o));
    }
    {   // mccg_solve: restrictions (tests/test_solvers.cpp:369-433 scenarios)
        struct M { int n, p; double cond; unsigned long long seed; double tol; bool dup; };
        const M ms[] = {{40, 3, 1e3, 37, 1e-6, false}, {30, 3, 1e2, 59, 1e-8, true}, {50, 8, 1e3, 5, 1e-9, false},
                        {40, 3, 1e2, 67, 1e-8, false}};
        for (const auto& c : ms) {
            ProblemSpec spec;
            spec.n = c.n;
            spec.p = c.p;
            spec.cond = c.cond;
            spec.seed = c.seed;
            auto inst = make_problem<double>(spec);
            if (c.dup)
                for (int i = 0; i < c.n; ++i) inst.X0(i, 2) = inst.X0(i, 1);
            SolveOptions<double> o;
            o.tol = c.tol;
            char name[96];
            std::snprintf(name, sizeof name, "mccg n=%d p=%d seed=%llu%s", c.n, c.p, c.seed, c.dup ? " dup" : "");
            compare(name, mccg_solve(inst.A, inst.b, inst.X0, o), gpu_mccg(inst.A, inst.b, inst.X0, o));
        }
    }
    {   // cg_solve / steepest_descent_solve through the p = 1 block kernels
        struct SCase { int n; double cond; unsigned long long seed; double tol; int max_iters; int recompute; };
        const SCase sc[] = {{120, 1e3, 21, 1e-10, -1, -1}, {120, 1e3, 21, 1e-10, -1, 0}, {80, 30.0, 22, 1e-9, -1, -1},
                            {64, 1e2, 5, 0.0, 25, 3}};
        for (const auto& c : sc) {
            ProblemSpec spec;
            spec.n = c.n;
            spec.p = 1;
            spec.cond = c.cond;
            spec.seed = c.seed;
            auto inst = make_problem<double>(spec);
            Vec<double> x0(inst.X0.col(0).begin(), inst.X0.col(0).end());
            SolveOptions<double> o;
            o.tol = c.tol;
            o.max_iters = c.max_iters;
            o.recompute_residual_every = c.recompute;
            char name[64];
            std::snprintf(name, sizeof name, "cg n=%d rec=%d", c.n, c.recompute);
            compare(name, cg_solve(inst.A, inst.b, x0, o), gpu_cg_solve(inst.A, inst.b, x0, o));
            std::snprintf(name, sizeof name, "steepest descent n=%d rec=%d", c.n, c.recompute);
            SolveOptions<double> os = o;
            if (os.max_iters < 0) os.max_iters = 400;
            compare(name, steepest_descent_solve(inst.A, inst.b, x0, os),
                    gpu_steepest_descent_solve(inst.A, inst.b, x0, os));
        }
    }
    {   // gpu_make_problem == make_problem<double>, field by field
        const ProblemSpec specs[] = {{2, 1, 3.0, 4}, {77, 3, 1e3, 9}, {300, 8, 1e4, 21}};
        for (const auto& spec : specs) {
            const auto r = make_problem<double>(spec);
            const auto g = gpu_make_problem(spec);
            bool ok = r.A == g.A && r.X0 == g.X0 && r.b.size() == g.b.size() && same(r.realized_cond, g.realized_cond);
            for (size_t i = 0; ok && i < r.b.size(); ++i) ok = same(r.b[i], g.b[i]);
            std::printf("gpu_make_problem n=%-4d p=%-2d        %s\n", spec.n, spec.p, ok ? "bit-identical" : "MISMATCH");
            if (!ok) ++failures;
        }
    }
    {   // error behaviour: indefinite matrix -> SpdViolationError; bad shapes -> DimensionError
        const int n = 30;
        std::vector<double> e(static_cast<size_t>(n) * n, 0.0);
        for (int i = 0; i < n; ++i) e[static_cast<size_t>(i) * n + i] = -1.0;
        SpdMatrix<double> A(n, e, SpdCheck::skip);
        Vec<double> b(n, 1.0);
        DenseBlock<double> X0(n, 2);
        for (int i = 0; i < n; ++i) X0(i, 1) = 0.01 * i;
        std::string ref_msg, gpu_msg;
        try { ccg_solve(A, b, X0, {}); } catch (const SpdViolationError& ex) { ref_msg = ex.what(); }
        try { gpu_ccg(A, b, X0, {}); } catch (const SpdViolationError& ex) { gpu_msg = ex.what(); }
        const bool ok = !ref_msg.empty() && ref_msg == gpu_msg;
        std::printf("%-34s %s (\"%s\")\n", "SpdViolationError", ok ? "same exception" : "MISMATCH", gpu_msg.c_str());
        if (!ok) ++failures;
        // gpu_mccg refuses the verification-only options instead of dropping them
        bool refused = false;
        SolveOptions<double> oh;
        oh.keep_history = true;
        try { gpu_mccg(A, b, X0, oh); } catch (const std::invalid_argument&) { refused = true; }
        std::printf("%-34s %s\n", "mccg keep_history refused", refused ? "invalid_argument" : "MISMATCH");
        if (!refused) ++failures;
        bool dim = false;
        try { gpu_ccg(A, Vec<double>(n - 1, 1.0), X0, {}); } catch (const DimensionError&) { dim = true; }
        std::printf("%-34s %s\n", "DimensionError", dim ? "same exception" : "MISMATCH");
        if (!dim) ++failures;
    }
    // Verification mode (trace.hpp:84-87): history blocks and A-norm errors, bit for bit
    // (the problem of tests/test_solvers.cpp:227-235, a tolerance run, recompute iterations, cg)
    {
        struct VCase { int n, p; double cond; unsigned long long seed; double tol; int max_iters; int recompute; };
        const VCase vc[] = {{60, 3, 100.0, 41, 1e-300, 15, -1}, {90, 4, 1e3, 5, 1e-9, -1, 4}, {70, 1, 1e2, 9, 1e-10, -1, 1}};
        for (const auto& c : vc) {
            ProblemSpec spec;
            spec.n = c.n;
            spec.p = c.p;
            spec.cond = c.cond;
            spec.seed = c.seed;
            auto inst = make_problem<double>(spec);
            const Vec<double> xs = solve_dense(inst.A, inst.b);
            SolveOptions<double> o;
            o.tol = c.tol;
            o.max_iters = c.max_iters;
            o.recompute_residual_every = c.recompute;
            o.keep_history = true;
            o.x_star = &xs;
            const auto r = ccg_solve(inst.A, inst.b, inst.X0, o);
            const auto g = gpu_ccg(inst.A, inst.b, inst.X0, o);
            char name[96];
            std::snprintf(name, sizeof name, "verify n=%d p=%d", c.n, c.p);
            compare(name, r, g);
            bool ok = r.history_x.size() == g.history_x.size() && r.history_r.size() == g.history_r.size() &&
                      r.history_d.size() == g.history_d.size() &&
                      g.history_x.size() == static_cast<size_t>(g.iteration_count()) + 1;
            for (size_t e = 0; ok && e < r.history_x.size(); ++e)
                ok = r.history_x[e] == g.history_x[e] && r.history_r[e] == g.history_r[e] &&
                     r.history_d[e] == g.history_d[e];
            for (int k = 0; ok && k < r.iteration_count(); ++k) {
                const auto& a = r.iterations[k].anorm_errors;
                const auto& bb = g.iterations[k].anorm_errors;
                ok = a.size() == bb.size() && a.size() == static_cast<size_t>(c.p);
                for (size_t j = 0; ok && j < a.size(); ++j) ok = same(a[j], bb[j]);
            }
            std::printf("%-34s entries=%zu  %s\n", "  history + anorm_errors", g.history_x.size(),
                        ok ? "bit-identical" : "MISMATCH");
            if (!ok) ++failures;
            if (c.p == 1) {  // the scalar solver keeps its own history / A-norm record (solvers.hpp:411-415, :489-504)
                Vec<double> x0(static_cast<size_t>(c.n));
                for (int i = 0; i < c.n; ++i) x0[static_cast<size_t>(i)] = inst.X0(i, 0);
                const auto rc = cg_solve(inst.A, inst.b, x0, o);
                const auto gc = gpu_cg_solve(inst.A, inst.b, x0, o);
                bool okc = rc.iteration_count() == gc.iteration_count() && rc.history_x.size() == gc.history_x.size();
                for (size_t e = 0; okc && e < rc.history_x.size(); ++e)
                    okc = rc.history_x[e] == gc.history_x[e] && rc.history_r[e] == gc.history_r[e] &&
                          rc.history_d[e] == gc.history_d[e];
                for (int k = 0; okc && k < rc.iteration_count(); ++k)
                    okc = rc.iterations[k].anorm_errors.size() == 1 && gc.iterations[k].anorm_errors.size() == 1 &&
                          same(rc.iterations[k].anorm_errors[0], gc.iterations[k].anorm_errors[0]);
                std::printf("%-34s entries=%zu  %s\n", "  cg_solve history + anorm", gc.history_x.size(),
                            okc ? "bit-identical" : "MISMATCH");
                if (!okc) ++failures;
            }
        }
    }
    std::printf("DROPIN %s (%d failures)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
