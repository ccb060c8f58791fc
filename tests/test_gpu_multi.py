"""Multi-GPU inside the library (include/coopcg_gpu.h).

coopcg_gpu_create_multi: one process drives several row shards; the kernel
that computes a shard's rows of Q stores them into every shard's Q (peer
stores; plain stores here, where the shards share this run's one GPU) and the
per-iteration exchange is a cross-stream event barrier enqueued by the
library's own run loop.  No kernel ever waits on another (the barrier is
stream ordering), so sharing one GPU is a faithful stand-in for the
ordering, and exact mode must be bit-identical to one context and to the
oracle for any split (the reference's operation order is per row,
kernels.hpp:28-34).

coopcg_gpu_create_rank: one process per GPU with NCCL row exchanges inside
the run loop; with one GPU only a world of one rank can run (NCCL refuses two
ranks on one device), which still drives the NCCL code path end to end.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    import paper_1204_0069_b200 as mod
    with mod.GpuContext(8, 2) as _:
        pass
    return mod


def _same(a, b):
    assert str(a.status) == str(b.status)
    assert a.iteration_count() == b.iteration_count()
    assert a.converged_agent == b.converged_agent
    assert np.array_equal(a.initial_residual_norms, b.initial_residual_norms)
    assert np.array_equal(a.residual_norms, b.residual_norms, equal_nan=True)
    assert np.array_equal(a.minres, b.minres)
    assert np.array_equal(a.final_x, b.final_x)
    assert np.array_equal(a.final_residual_norms, b.final_residual_norms)


@pytest.mark.parametrize("n,p,ndev,matrix,max_iters,recompute", [
    (600, 4, 2, "householder", -1, -1),
    (517, 8, 3, "diagdom", 60, -1),       # post-convergence tail, a recompute at k = 49
    (256, 16, 2, "diagdom", 55, 7),       # R exchanged every 7th iteration
    (1000, 3, 4, "diagdom", -1, -1),      # config 0 over four shards
    (300, 32, 2, "householder", 30, -1),
])
def test_multi_exact_bitwise(m, po, n, p, ndev, matrix, max_iters, recompute):
    A = po.gen_diagdom(n, n) if matrix == "diagdom" else po.gen_householder(n, 8, 1e3, n)
    b = po.gen_rhs(n, "uniform", n)
    X0 = po.gen_starts(n, p, n)
    tol = 1e-10 * po.seq_norm(b) if max_iters < 0 else 0.0
    opts = m.SolveOptions(tol=tol, max_iters=max_iters, recompute_residual_every=recompute)
    with m.GpuContext(n, p, devices=[0] * ndev) as g:
        assert len(g.shards()) == ndev
        assert [r for _, r, _ in g.shards()][0] == 0 and g.shards()[-1][2] == n
        g.set_A(A)
        gt = g.solve(b, X0, opts)
        t2 = g.solve(b, X0, opts)  # resident A: deterministic
    one = m.ccg_solve(A, b, X0, opts)
    ot = po.oracle_ccg(A, b, X0, tol=tol, max_iters=max_iters, recompute=recompute)
    _same(gt, one)
    _same(gt, t2)
    assert str(gt.status) == ot.status and gt.iteration_count() == ot.iterations
    assert np.array_equal(gt.residual_norms, ot.residual_norms)
    assert np.array_equal(gt.final_x, ot.final_x)
    assert np.array_equal(gt.final_residual_norms, ot.final_residual_norms)


def test_multi_generators_and_row_calls(m, po):
    n, p = 700, 4
    with m.GpuContext(n, p, devices=[0, 0, 0]) as g:
        g.gen_A("householder", 31, 8, 1e4)
        A = g.get_A()
        assert np.array_equal(A, po.gen_householder(n, 8, 1e4, 31))
        assert np.array_equal(g.get_A(250, 300), A[250:550])   # spans two shards
        D = np.random.default_rng(2).uniform(-1, 1, (n, p))
        ref = np.zeros((p, n))
        Dc = np.ascontiguousarray(D.T)
        po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, ref.ctypes.data)
        assert np.array_equal(g.matvec_block(D), ref.T)
        g.gen_A("diagdom", 32)
        assert np.array_equal(g.get_A(), po.gen_diagdom(n, 32))
        b = po.gen_rhs(n, "uniform", 32)
        X0 = po.gen_starts(n, p, 32)
        gt = g.solve(b, X0, m.SolveOptions(tol=1e-10 * po.seq_norm(b)))
    ot = po.oracle_ccg(po.gen_diagdom(n, 32), b, X0, tol=1e-10 * po.seq_norm(b))
    assert np.array_equal(gt.final_x, ot.final_x) and np.array_equal(gt.residual_norms, ot.residual_norms)


def test_multi_mccg_restriction(m, po):
    n, p = 240, 6
    A = po.gen_householder(n, 6, 1e3, 11)
    b = po.gen_rhs(n, "normal", 11)
    X0 = po.gen_starts(n, p, 11)
    X0[:, 4] = X0[:, 2]
    X0[:, 5] = X0[:, 1]
    tol = 1e-9 * po.seq_norm(b)
    with m.GpuContext(n, p, devices=[0, 0]) as g:
        g.set_A(A)
        gt = g.solve(b, X0, m.SolveOptions(tol=tol, algo="mccg"))
    ot = po.oracle_ccg(A, b, X0, tol=tol, algo="mccg")
    assert gt.active_agents == ot.extra["active_agents"]
    assert np.array_equal(gt.residual_norms, ot.residual_norms, equal_nan=True)
    assert np.array_equal(gt.final_x, ot.final_x[:, gt.active_agents])


@pytest.mark.parametrize("n,p,ndev", [(1000, 3, 2), (900, 16, 3)])
def test_multi_fast_within_tolerance(m, po, n, p, ndev):
    A = po.gen_diagdom(n, n + 1)
    b = po.gen_rhs(n, "uniform", n + 1)
    X0 = po.gen_starts(n, p, n + 1)
    tol = 1e-10 * po.seq_norm(b)
    gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=tol), m.GpuOptions(arith="fast", devices=[0] * ndev))
    ot = po.oracle_ccg(A, b, X0, tol=tol)
    assert str(gt.status) == "converged" and abs(gt.iteration_count() - ot.iterations) <= 2
    rel = np.linalg.norm(gt.final_x - ot.final_x, axis=0) / np.linalg.norm(ot.final_x, axis=0)
    assert rel.max() < 1e-8


@pytest.mark.parametrize("n,p,ndev,m_refl,kappa,recompute", [(288, 4, 2, 3, 3.3e3, -1), (288, 4, 3, 3, 3.3e3, -1),
                                                             (513, 9, 3, 8, 4.5e2, 0)])
def test_multi_fast_long_run_on_unequal_shards(m, po, n, p, ndev, m_refl, kappa, recompute):
    """Fast mode over UNEQUAL row shards for hundreds of iterations (a case of
    tools/fuzz_parity.py): every shard must sum the replicated Grams in the same
    grouping, or alpha / beta -- and with them the replicated X, R, D -- drift
    apart between the shards and the solve diverges after ~20 iterations (the
    row-pass grid used to depend on the shard's own row count)."""
    A = po.gen_householder(n, m_refl, kappa, 1600630417)
    b = po.gen_rhs(n, "normal", 1600630417)
    X0 = po.gen_starts(n, p, 1600630417)
    tol = 2.4e-10 * po.seq_norm(b)
    opts = m.SolveOptions(tol=tol, recompute_residual_every=recompute)
    ref = po.oracle_ccg(A, b, X0, tol=tol, recompute=recompute)
    one = m.ccg_solve(A, b, X0, opts, m.GpuOptions(arith="fast"))
    gt = m.ccg_solve(A, b, X0, opts, m.GpuOptions(arith="fast", devices=[0] * ndev))
    assert ref.status == "converged" and ref.iterations > 60
    assert str(one.status) == str(gt.status) == "converged"
    assert abs(gt.iteration_count() - ref.iterations) <= max(4, ref.iterations // 20)
    assert abs(one.iteration_count() - ref.iterations) <= max(4, ref.iterations // 20)
    rel = np.linalg.norm(gt.final_x - ref.final_x, axis=0) / np.linalg.norm(ref.final_x, axis=0)
    assert rel.max() < 10 * kappa * 2.4e-10  # both within kappa * tol of the solution
    again = m.ccg_solve(A, b, X0, opts, m.GpuOptions(arith="fast", devices=[0] * ndev))
    assert np.array_equal(again.residual_norms, gt.residual_norms)  # deterministic


def test_multi_rejects_bad_splits(m):
    with pytest.raises(m.DimensionError):
        m.GpuContext(3, 1, devices=[0, 0, 0, 0])
    with m.GpuContext(200, 2, devices=[0, 0]) as g:
        with pytest.raises(m.Error, match="multi-device handle"):
            m.solver._check(g._h, m.solver._capi.lib().coopcg_gpu_begin(g._h, None))


def test_rank_context_nccl_world_of_one(m, po):
    """coopcg_gpu_create_rank with nranks = 1: the NCCL exchange path of the
    run loop (grouped broadcasts) on this GPU, bit-identical to the oracle."""
    n, p = 512, 8
    uid = m.nccl_unique_id()
    with m.GpuContext(n, p, nccl=(1, 0, uid)) as r:
        assert (r.row_begin, r.row_end) == (0, n)
        r.gen_A("householder", 9, 8, 1e3)
        A = r.get_A()
        assert np.array_equal(A, po.gen_householder(n, 8, 1e3, 9))
        b = po.gen_rhs(n, "normal", 9)
        X0 = po.gen_starts(n, p, 9)
        gt = r.solve(b, X0, m.SolveOptions(max_iters=60, recompute_residual_every=9))
    ot = po.oracle_ccg(A, b, X0, max_iters=60, recompute=9)
    assert np.array_equal(gt.residual_norms, ot.residual_norms)
    assert np.array_equal(gt.final_x, ot.final_x)


def test_row_split_covers_the_rows(m):
    for n, parts in ((1000, 3), (131072, 8), (65536, 8), (100, 7), (64, 2)):
        rows = [m.row_split(n, parts, g) for g in range(parts)]
        assert rows[0][0] == 0 and rows[-1][1] == n
        assert all(rows[g][1] == rows[g + 1][0] for g in range(parts - 1))
