"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and the oracle, bit for bit (exact mode).

Mirrors the reference's hot-path tests: matvec_block == naive
loop bitwise (tests/test_dense.cpp:82-86), numerical_rank cases
(test_dense.cpp:246-291), degenerate start => RankCollapse at k = 0
(test_solvers.cpp:369-385), identity converges in one iteration
(test_solvers.cpp:203-212), recompute policies (test_solvers.cpp:176-201),
concurrent independent solves (test_parallel.cpp:190-204)."""
import threading

import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_1204_0069_b200 as mod
    # Fail loudly (never skip) when the CUDA path is unavailable on a GPU box.
    with mod.GpuContext(8, 2) as _:
        pass
    return mod


def assert_same(gt, ot):
    """gt: product SolveTrace, ot: oracle/reference trace (pyoracle.Trace)."""
    assert str(gt.status) == ot.status
    assert gt.iteration_count() == ot.iterations
    assert gt.converged_agent == ot.converged_agent
    assert np.array_equal(gt.initial_residual_norms, ot.initial_residual_norms)
    assert np.array_equal(gt.residual_norms, ot.residual_norms)
    assert np.array_equal(gt.minres, ot.minres)
    assert np.array_equal(gt.final_x, ot.final_x)
    assert np.array_equal(gt.final_residual_norms, ot.final_residual_norms)
    assert gt.final_minres == ot.final_minres


@pytest.mark.parametrize("name", golden_names())
def test_golden_bitwise(m, name):
    A, z = load_golden(name)
    algo = str(z["algo"]) if "algo" in z else "ccg"
    if algo in ("cg", "sd"):
        fn = m.cg_solve if algo == "cg" else m.steepest_descent_solve
        t = fn(A, z["b"], z["X0"][:, 0], m.SolveOptions(tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                                                          recompute_residual_every=int(z["recompute"])))
        assert str(t.status) == str(z["status"]) and t.iteration_count() == int(z["iterations"])
        assert np.array_equal(t.residual_norms, z["residual_norms"])
        assert np.array_equal(t.final_x, z["final_x"])
        assert np.array_equal(t.final_residual_norms, z["final_residual_norms"])
        return
    opts = m.SolveOptions(tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                          recompute_residual_every=int(z["recompute"]), algo=algo)
    if int(z["rc"]) == 2:
        with pytest.raises(m.SpdViolationError, match="nonpositive direction energy"):
            m.ccg_solve(A, z["b"], z["X0"], opts)
        return
    if int(z["rc"]) == 3:
        with pytest.raises(m.NumericalBreakdownError, match="numerically zero|degenerate"):
            m.ccg_solve(A, z["b"], z["X0"], opts)
        return
    t = m.ccg_solve(A, z["b"], z["X0"], opts)
    assert str(t.status) == str(z["status"])
    assert t.iteration_count() == int(z["iterations"])
    assert t.converged_agent == int(z["converged_agent"])
    assert np.array_equal(t.residual_norms, z["residual_norms"], equal_nan=True)
    assert np.array_equal(t.minres, z["minres"])
    assert np.array_equal(t.initial_residual_norms, z["initial_residual_norms"])
    act = t.active_agents
    assert act == ([int(a) for a in z["active_agents"]] if len(z["active_agents"]) else act)
    assert np.array_equal(t.final_x, z["final_x"][:, act])
    assert np.array_equal(t.final_residual_norms_by_id, z["final_residual_norms"], equal_nan=True)


CASES = [  # (n, p, matrix, tol_rel, max_iters, recompute)
    (1000, 3, "diagdom", 1e-10, -1, -1),      # cfg 0 itself
    (333, 1, "diagdom", 1e-12, -1, -1),
    (257, 5, "householder", 1e-10, -1, -1),   # padded P (5 -> 8), ragged tiles
    (512, 8, "diagdom", 0.0, 120, -1),        # post-convergence tail + recomputes
    (384, 16, "householder", 0.0, 60, 7),
    (640, 32, "diagdom", 0.0, 40, -1),
    (200, 12, "householder", 1e-9, -1, 1),    # recompute every iteration
    (199, 4, "householder", 1e-9, -1, 0),     # never recompute
]


@pytest.mark.parametrize("n,p,matrix,tol_rel,max_iters,recompute", CASES)
def test_vs_oracle_bitwise(m, po, n, p, matrix, tol_rel, max_iters, recompute):
    seed = n * 31 + p
    A = po.gen_diagdom(n, seed) if matrix == "diagdom" else po.gen_householder(n, 8, 1e4, seed)
    b = po.gen_rhs(n, "uniform" if matrix == "diagdom" else "normal", seed)
    X0 = po.gen_starts(n, p, seed)
    tol = tol_rel * po.seq_norm(b)
    ot = po.oracle_ccg(A, b, X0, tol=tol, max_iters=max_iters, recompute=recompute)
    gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=tol, max_iters=max_iters,
                                              recompute_residual_every=recompute))
    assert_same(gt, ot)


def test_device_generators_match_oracle(m, po):
    with m.GpuContext(300, 3) as ctx:
        ctx.gen_A("diagdom", 77)
        assert np.array_equal(ctx.get_A(), po.gen_diagdom(300, 77))
    with m.GpuContext(256, 4) as ctx:
        ctx.gen_A("householder", 78, 8, 1e4)
        assert np.array_equal(ctx.get_A(), po.gen_householder(256, 8, 1e4, 78))


def test_generated_problem_solves_like_oracle(m, po):
    cfg = m.CONFIGS[0]
    with m.GpuContext(cfg.n, cfg.p) as ctx:
        b, X0, opts = m.make_problem_on_device(ctx, cfg)
        gt = ctx.solve(b, X0, opts)
    A = po.gen_diagdom(cfg.n, cfg.seed)
    ot = po.oracle_ccg(A, b, X0, tol=opts.tol, max_iters=opts.max_iters)
    assert_same(gt, ot)
    assert str(gt.status) == "converged"


# n >= 148 * 64 selects 64-row panels (and two rows per thread at P >= 16),
# n > 148 * 64 at P = 8 the 128-row panels of the pipelined kernel, as at
# P = 16 (ad_exact_pipe_kernel): the A.D configurations of BASELINE configs
# 2-4 (coopcg_gpu.cu pick_ad_config).  12345: partial last panel, partial
# last k-tile and an odd k count (masked last batch).
@pytest.mark.parametrize("n,p", [(1000, 3), (777, 17), (96, 32), (130, 1),
                                 (9472, 8), (9473, 8), (12345, 7), (9473, 16), (9500, 24)])
def test_matvec_block_bitwise(m, po, n, p):
    rng = np.random.default_rng(n + p)
    A = po.gen_diagdom(n, 5) if n < 2000 else rng.uniform(-1, 1, (n, n))
    A[3, :] *= 1.5  # non-symmetric input: the device layout must still follow A's rows
    D = rng.uniform(-1, 1, (n, p))
    ref = np.zeros((p, n))
    Dc = np.ascontiguousarray(D.T)
    po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, ref.ctypes.data)
    with m.GpuContext(n, p) as ctx:
        ctx.set_A(A)
        out = ctx.matvec_block(D)
    assert np.array_equal(out, ref.T)


def test_matvec_block_shard_rows_pipelined(m, po):
    """A row shard large enough for the pipelined A.D (n_loc > 9472 at P = 8)
    starting at a nonzero row offset, next to a small shard."""
    n, p = 10007, 8
    rng = np.random.default_rng(11)
    A = rng.uniform(-1, 1, (n, n))
    D = rng.uniform(-1, 1, (n, p))
    ref = np.zeros((p, n))
    Dc = np.ascontiguousarray(D.T)
    po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, ref.ctypes.data)
    for r0, r1 in ((0, 407), (407, n)):
        with m.GpuContext(n, p, row_begin=r0, row_end=r1) as ctx:
            ctx.set_A(A[r0:r1])
            out = ctx.matvec_block(D)
        assert np.array_equal(out, ref.T[r0:r1])


def test_pipelined_ad_solve_bitwise(m, po):
    """A few exact iterations (with a residual recompute) on the pipelined A.D
    path (n > 9472, p = 8): identical to the oracle."""
    n, p = 9601, 8
    A = po.gen_diagdom(n, 21)
    b = po.gen_rhs(n, "uniform", 21)
    X0 = po.gen_starts(n, p, 21)
    ot = po.oracle_ccg(A, b, X0, tol=0.0, max_iters=6, recompute=4)
    gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=0.0, max_iters=6, recompute_residual_every=4))
    assert_same(gt, ot)


def test_matvec_block_shard_rows(m, po):
    n, p = 500, 4
    A = po.gen_diagdom(n, 6)
    D = np.random.default_rng(1).uniform(-1, 1, (n, p))
    ref = np.zeros((p, n))
    Dc = np.ascontiguousarray(D.T)
    po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, ref.ctypes.data)
    for r0, r1 in ((0, 137), (137, 300), (300, 500)):
        with m.GpuContext(n, p, row_begin=r0, row_end=r1) as ctx:
            ctx.set_A(A[r0:r1])
            assert np.array_equal(ctx.matvec_block(D), ref.T[r0:r1])


def _rank_blocks(n):
    rng = np.random.default_rng(3)
    v, w, u = rng.uniform(-1, 1, (3, n))
    return {
        "full": rng.uniform(-1, 1, (n, 4)),
        "v_2v_w": np.stack([v, 2 * v, w, u], 1),
        "zero": np.zeros((n, 4)),
        "near": np.stack([v, v + 1e-13 * w, w, u], 1),
        "scaled": np.stack([v * 1e-150, w, u, v + w], 1),
        "permuted": np.stack([w, u, v, 2 * v], 1),
    }


@pytest.mark.parametrize("force_exact", [False, True])
def test_numerical_rank_matches_oracle(m, po, force_exact):
    n = 300
    with m.GpuContext(n, 4) as ctx:
        for name, blk in _rank_blocks(n).items():
            expect = po.numerical_rank(blk, 1e-10)[0]
            got = ctx.numerical_rank(blk, 1e-10, force_exact=force_exact)
            assert got == expect, name


def test_degenerate_start_rank_collapse(m, po):
    n = 200
    A = po.gen_diagdom(n, 2)
    b = po.gen_rhs(n, "uniform", 2)
    t = m.ccg_solve(A, b, np.zeros((n, 3)), m.SolveOptions(tol=1e-10))
    assert str(t.status) == "rank-collapse" and t.iteration_count() == 0


def test_max_iters_zero_and_converged_at_setup(m, po):
    n = 120
    A = po.gen_diagdom(n, 3)
    b = po.gen_rhs(n, "uniform", 3)
    X0 = po.gen_starts(n, 3, 3)
    for opts in (m.SolveOptions(max_iters=0), m.SolveOptions(tol=1e6)):
        gt = m.ccg_solve(A, b, X0, opts)
        ot = po.oracle_ccg(A, b, X0, tol=opts.tol, max_iters=opts.max_iters)
        assert_same(gt, ot)
        assert gt.iteration_count() == 0


def test_concurrent_contexts_are_independent(m, po):
    n, p = 400, 4
    A = po.gen_householder(n, 8, 1e3, 4)
    b = po.gen_rhs(n, "normal", 4)
    X0 = po.gen_starts(n, p, 4)
    opts = m.SolveOptions(tol=1e-9 * po.seq_norm(b))
    out = [None] * 4

    def work(i):
        out[i] = m.ccg_solve(A, b, X0, opts)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    for t in out[1:]:
        assert np.array_equal(t.final_x, out[0].final_x)
        assert np.array_equal(t.residual_norms, out[0].residual_norms)


def test_resident_reuse_is_deterministic(m, po):
    """Two runs on one context (resident A) give identical bytes."""
    n, p = 600, 8
    with m.GpuContext(n, p) as ctx:
        ctx.gen_A("diagdom", 9)
        b = m.gen_rhs(n, "uniform", 9)
        X0 = m.gen_starts(n, p, 9)
        t1 = ctx.solve(b, X0, m.SolveOptions(max_iters=70))
        t2 = ctx.solve(b, X0, m.SolveOptions(max_iters=70))
    assert np.array_equal(t1.final_x, t2.final_x)
    assert np.array_equal(t1.residual_norms, t2.residual_norms)


def test_scalar_solvers_raise_the_reference_texts(m):
    """cg_solve / steepest_descent_solve on an indefinite matrix: SpdViolationError
    with the scalar solvers' own messages (solvers.hpp:448-449, :583-585)."""
    n = 24
    A = -np.eye(n)
    b = np.ones(n)
    x0 = np.linspace(0.0, 1.0, n)
    with pytest.raises(m.SpdViolationError, match=r"^cg_solve: nonpositive direction energy at iteration 0$"):
        m.cg_solve(A, b, x0)
    with pytest.raises(m.SpdViolationError,
                       match=r"^steepest_descent_solve: nonpositive gradient energy at iteration 0$"):
        m.steepest_descent_solve(A, b, x0)
