"""Verification mode of the solvers (SolveOptions.keep_history / x_star,
coopcg/trace.hpp:84-87) on the GPU backend.

The reference uses it for its own invariant tests (tests/test_solvers.cpp:227-295:
orthogonality of residual blocks, conjugacy of direction blocks, optimality,
monotone objective and A-norm error); this file restates those checks for the
device solver in both arithmetic modes, pins the A-norm errors bit for bit
against a sequential pure-Python restatement of a_norm (dense_ops.hpp:159-196,
block_cg.hpp:316-331), and checks the history blocks against the solve they
belong to.  The bit-for-bit comparison of history_x / _r / _d and anorm_errors
with the reference's own ccg_solve / cg_solve runs through the C++ drop-in
(oracle/dropin_test.cpp, tests/test_gpu_dropin.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_1204_0069_b200 as mod
    return mod


def seq_dot(a, b):
    acc = np.float64(0.0)
    for x, y in zip(a, b):
        acc = acc + x * y  # separately rounded product and sum (kernels.hpp:20-26)
    return acc


def seq_anorm(A, diff):
    ax = np.array([seq_dot(A[i], diff) for i in range(A.shape[0])])
    q = seq_dot(diff, ax)
    return float(np.sqrt(q)) if q >= 0 else 0.0


def problem(m, n, p, cond, seed, arith):
    ctx = m.GpuContext(n, p, arith=arith)
    b, X0 = m.make_reference_problem_on_device(ctx, cond, seed)
    A = ctx.get_A()
    xs = np.linalg.solve(A, b)
    return ctx, A, b, X0, xs


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_history_invariants(m, arith):
    """tests/test_solvers.cpp:227-295 on the device solver."""
    n, p = 60, 3
    ctx, A, b, X0, xs = problem(m, n, p, 100.0, 41, arith)
    with ctx:
        t = ctx.solve(b, X0, m.SolveOptions(tol=1e-300, max_iters=15, keep_history=True, x_star=xs))
    assert t.iteration_count() == 15
    hx, hr, hd = t.history_x, t.history_r, t.history_d
    assert len(hx) == len(hr) == len(hd) == 16
    assert np.array_equal(hx[0], X0) and np.array_equal(hx[-1], t.final_x)
    assert np.array_equal(hd[0], hr[0])  # D0 = R0 (block_cg.hpp:139-144)
    # residual blocks mutually orthogonal
    scale_r = max(float(np.max(np.sum(r * r, axis=0))) for r in hr)
    for i in range(len(hr)):
        for j in range(i + 1, len(hr)):
            assert np.max(np.abs(hr[i].T @ hr[j])) <= 1e-10 * scale_r, (i, j)
    # direction blocks mutually A-conjugate
    had = [A @ d for d in hd]
    scale_d = max(float(np.max(np.abs(np.sum(d * ad, axis=0)))) for d, ad in zip(hd, had))
    for i in range(len(hd)):
        for j in range(i + 1, len(hd)):
            assert np.max(np.abs(hd[i].T @ had[j])) <= 1e-10 * scale_d, (i, j)
    # optimality: earlier directions are orthogonal to every agent's current gradient
    for k in range(1, len(hx)):
        grad = A @ hx[k] - b[:, None]
        for i in range(k):
            assert np.max(np.abs(hd[i].T @ grad)) <= 1e-8 * scale_d, (k, i)
    # monotone objective per agent
    f = [0.5 * np.sum(x * (A @ x), axis=0) - b @ x for x in hx]
    for k in range(1, len(f)):
        assert np.all(f[k] <= f[k - 1] + 1e-9 * (1.0 + np.abs(f[k - 1])))
    # recorded A-norm errors nonincreasing, and the recorded values are a_norm(x_j - x*)
    an = np.array([rec.anorm_errors for rec in t.iterations])
    assert an.shape == (15, p)
    assert np.all(an[1:] <= an[:-1] * (1.0 + 1e-9))
    for k in (0, 7, 14):
        for j in range(p):
            want = seq_anorm(A, hx[k + 1][:, j] - xs)
            if arith == "exact":
                assert an[k, j] == want, (k, j)  # same operation sequence: same bits
            else:
                assert abs(an[k, j] - want) <= 1e-9 * max(want, 1e-300) + 1e-13 * an[0, j], (k, j)
    # stored recurrence residual against the recomputed one (tests/test_solvers.cpp:435-456)
    for k in range(len(hx)):
        assert np.max(np.abs(hr[k] - (A @ hx[k] - b[:, None]))) <= 1e-8 * np.linalg.norm(b)


def test_history_follows_the_stop_and_recompute_iterations(m, po):
    """A tolerance run: entries = iterations + 1, the last entry is the final
    state, and the run is the same solve bit for bit with and without the
    verification mode (recompute iterations included)."""
    n, p = 300, 4
    with m.GpuContext(n, p) as ctx:  # the cfg-0 family: converges in about ten iterations
        ctx.gen_A("diagdom", 5)
        A = ctx.get_A()
        b = m.gen_rhs(n, "uniform", 5)
        X0 = m.gen_starts(n, p, 5)
        xs = np.linalg.solve(A, b)
        tol = 1e-10 * float(np.linalg.norm(b))
        opts = m.SolveOptions(tol=tol, recompute_residual_every=4)
        plain = ctx.solve(b, X0, opts)
        t = ctx.solve(b, X0, m.SolveOptions(tol=tol, recompute_residual_every=4, keep_history=True, x_star=xs))
        again = ctx.solve(b, X0, opts)  # verification switched off again on the same context
    ref = po.oracle_ccg(A, b, X0, tol=tol, max_iters=-1, recompute=4)
    assert t.iteration_count() > 4
    assert str(t.status) == ref.status == "converged" and t.iteration_count() == ref.iterations
    for s in (plain, t, again):
        assert np.array_equal(s.residual_norms, ref.residual_norms) and np.array_equal(s.final_x, ref.final_x)
    assert len(t.history_x) == t.iteration_count() + 1
    assert np.array_equal(t.history_x[-1], t.final_x)
    assert not plain.history_x and not again.history_x and again.iterations[0].anorm_errors is None
    # recorded norms are the norms of the stored residual blocks
    for k, rec in enumerate(t.iterations):
        got = np.sqrt(np.sum(t.history_r[k + 1] ** 2, axis=0))
        assert np.allclose(got, rec.residual_norms, rtol=1e-12, atol=0)
    j = t.converged_agent
    assert t.iterations[-1].anorm_errors[j] == seq_anorm(A, t.final_x[:, j] - xs)
    # the converging iteration's direction block: Dnext = R + D beta^T is formed before the
    # stop (solvers.hpp:146), so it is conjugate to the previous direction block
    d_last, d_prev = t.history_d[-1], t.history_d[-2]
    scale = float(np.max(np.abs(np.sum(d_prev * (A @ d_prev), axis=0))))
    assert np.max(np.abs(d_last.T @ (A @ d_prev))) <= 1e-8 * scale
    assert not np.array_equal(d_last, d_prev)


def test_scalar_cg_records_anorm(m):
    """cg_solve with x_star (solvers.hpp:489-494): the classical CG error bound
    2 ((sqrt(kappa) - 1) / (sqrt(kappa) + 1))^k of tests/test_solvers.cpp:297-320."""
    n = 80
    ctx, A, b, X0, xs = problem(m, n, 1, 1e4, 43, "exact")
    ctx.close()
    t = m.cg_solve(A, b, X0[:, 0], m.SolveOptions(tol=1e-10, x_star=xs))
    e0 = seq_anorm(A, X0[:, 0] - xs)
    rho = (np.sqrt(1e4) - 1.0) / (np.sqrt(1e4) + 1.0)
    for rec in t.iterations:
        assert rec.anorm_errors.shape == (1,)
        assert rec.anorm_errors[0] <= 2.0 * rho ** (rec.k + 1) * e0 * (1.0 + 1e-8)


def test_verification_mode_is_refused_where_it_does_not_apply(m):
    n, p = 64, 3
    with m.GpuContext(n, p) as ctx:
        b, X0 = m.make_reference_problem_on_device(ctx, 10.0, 3)
        with pytest.raises(m.Error):  # mccg_solve restricts the blocks: not carried
            ctx.solve(b, X0, m.SolveOptions(tol=1e-8, algo="mccg", keep_history=True))
        with pytest.raises(m.DimensionError):
            ctx.solve(b, X0, m.SolveOptions(tol=1e-8, x_star=np.zeros(n + 1)))
        t = ctx.solve(b, X0, m.SolveOptions(tol=1e-8))  # the context still solves
        assert str(t.status) == "converged"
    with m.GpuContext(n, p, devices=[0, 0]) as ctx:  # row shards: one context must hold every row
        ctx.gen_A("diagdom", 3)
        b = m.gen_rhs(n, "uniform", 3)
        X0 = m.gen_starts(n, p, 3)
        with pytest.raises(m.Error):
            ctx.solve(b, X0, m.SolveOptions(tol=1e-8, keep_history=True))
