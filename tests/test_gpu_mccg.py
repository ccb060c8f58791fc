"""mccg_solve on the GPU (restriction on rank drop, solvers.hpp:156-175):
bit-identical to the oracle restatement, which tests/test_oracle.py pins to
the reference's mccg_solve (golden fixtures mccg_*)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cmp(m, po, A, b, X0, **kw):
    ot = po.oracle_ccg(A, b, X0, algo="mccg", **kw)
    gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=kw.get("tol", 0.0), max_iters=kw.get("max_iters", -1),
                                              recompute_residual_every=kw.get("recompute", -1), algo="mccg"))
    assert str(gt.status) == ot.status and gt.iteration_count() == ot.iterations
    assert gt.converged_agent == ot.converged_agent
    assert np.array_equal(gt.residual_norms, ot.residual_norms, equal_nan=True)
    assert gt.active_agents == ot.extra["active_agents"]
    assert np.array_equal(gt.final_x, ot.final_x[:, gt.active_agents])
    assert np.array_equal(gt.final_residual_norms_by_id, ot.final_residual_norms, equal_nan=True)
    return gt


@pytest.mark.parametrize("n,p,kind,seed,tol", [
    (300, 3, "dd", 3, 1e-10),          # full rank: mccg == ccg
    (120, 6, "hh", 4, 1e-13),          # Householder family, tight tolerance (converges before any
    (96, 8, "hh", 7, 1e-14),           # rank drop; restrictions: the golden mccg_* fixtures in
                                       # test_gpu_parity and the duplicate-column case below)
])
def test_mccg_vs_oracle(po, n, p, kind, seed, tol):
    import paper_1204_0069_b200 as m
    A = po.gen_diagdom(n, seed) if kind == "dd" else po.gen_householder(n, 6, 1e3, seed)
    b = po.gen_rhs(n, "uniform", seed)
    X0 = po.gen_starts(n, p, seed)
    _cmp(m, po, A, b, X0, tol=tol * po.seq_norm(b))


def test_mccg_duplicate_start_columns(po):
    import paper_1204_0069_b200 as m
    n, p = 200, 4
    A = po.gen_householder(n, 6, 1e3, 9)
    b = po.gen_rhs(n, "normal", 9)
    X0 = po.gen_starts(n, p, 9)
    X0[:, 3] = X0[:, 1]   # rank(D0) = 3: restricted at setup
    gt = _cmp(m, po, A, b, X0, tol=1e-9 * po.seq_norm(b))
    assert gt.iterations[0].active_agents == 3 and 3 not in gt.iterations[0].agents


def test_mccg_resident_context_resets_between_solves(po):
    """A restricted solve must not leak its reduced agent count into the next."""
    import paper_1204_0069_b200 as m
    n, p = 200, 4
    A = po.gen_householder(n, 6, 1e3, 9)
    b = po.gen_rhs(n, "normal", 9)
    X0 = po.gen_starts(n, p, 9)
    Xd = X0.copy()
    Xd[:, 3] = Xd[:, 1]
    with m.GpuContext(n, p) as ctx:
        ctx.set_A(A)
        t1 = ctx.solve(b, Xd, m.SolveOptions(tol=1e-9, algo="mccg"))
        t2 = ctx.solve(b, X0, m.SolveOptions(tol=1e-9))
    ref = po.oracle_ccg(A, b, X0, tol=1e-9)
    assert len(t1.active_agents) < p
    assert np.array_equal(t2.final_x, ref.final_x) and np.array_equal(t2.residual_norms, ref.residual_norms)


def test_mccg_fast_mode_converges(po):
    import paper_1204_0069_b200 as m
    n, p = 300, 4
    A = po.gen_householder(n, 6, 1e3, 9)
    b = po.gen_rhs(n, "normal", 9)
    X0 = po.gen_starts(n, p, 9)
    X0[:, 3] = X0[:, 1]
    t = m.ccg_solve(A, b, X0, m.SolveOptions(tol=1e-9 * po.seq_norm(b), algo="mccg"), m.GpuOptions(arith="fast"))
    ot = po.oracle_ccg(A, b, X0, tol=1e-9 * po.seq_norm(b), algo="mccg")
    assert str(t.status) == "converged" and t.active_agents == ot.extra["active_agents"]
    rel = np.linalg.norm(t.final_x - ot.final_x[:, t.active_agents], axis=0) / np.linalg.norm(t.final_x, axis=0)
    assert rel.max() < 1e-8


def test_mccg_restricted_then_larger_trace(po):
    """after a restricted mccg solve the next solve on the
    same context asks for a larger trace; the trace buffers must be sized for
    the context's original agent count, not the restricted one."""
    import paper_1204_0069_b200 as m
    n, p = 240, 6
    A = po.gen_householder(n, 6, 1e3, 11)
    b = po.gen_rhs(n, "normal", 11)
    X0 = po.gen_starts(n, p, 11)
    Xd = X0.copy()
    Xd[:, 4] = Xd[:, 2]
    Xd[:, 5] = Xd[:, 1]   # rank(D0) = 4: restricted at setup
    with m.GpuContext(n, p) as ctx:
        ctx.set_A(A)
        t1 = ctx.solve(b, Xd, m.SolveOptions(tol=0.0, max_iters=3, algo="mccg"))
        assert len(t1.active_agents) == 4
        t2 = ctx.solve(b, X0, m.SolveOptions(tol=1e-9 * po.seq_norm(b)))   # 2n-row trace
        t3 = ctx.solve(b, Xd, m.SolveOptions(tol=1e-9 * po.seq_norm(b), max_iters=3 * n, algo="mccg"))
    ref = po.oracle_ccg(A, b, X0, tol=1e-9 * po.seq_norm(b))
    assert t2.iteration_count() == ref.iterations
    assert np.array_equal(t2.final_x, ref.final_x) and np.array_equal(t2.residual_norms, ref.residual_norms)
    ref3 = po.oracle_ccg(A, b, Xd, tol=1e-9 * po.seq_norm(b), max_iters=3 * n, algo="mccg")
    assert np.array_equal(t3.residual_norms, ref3.residual_norms, equal_nan=True)
    assert np.array_equal(t3.final_x, ref3.final_x[:, t3.active_agents])
