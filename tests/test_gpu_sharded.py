"""The row-sharded phase API of the CUDA library (include/coopcg_gpu.h) with
two shard contexts on one GPU, exchanged in-process in lockstep (host-driven
copies between phases; no kernel ever waits on another).  Exact mode must be
bit-identical to the single-context solve and to the oracle; fast mode within
the fast-mode tolerances."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1204_0069_b200.sharded import (BLOCK_Q, BLOCK_R, BLOCK_S, PH_FINAL_LOCAL, PH_FINAL_REST, PH_ITER_LOCAL,
                                          PH_ITER_MID, PH_ITER_REST, PH_MCCG_SETUP, PH_SETUP_LOCAL, PH_SETUP_REST,
                                          GpuShardEngine)


def exchange(engines, which, k):
    torch.cuda.synchronize()
    blocks = [e.block(which, k) for e in engines]
    for i, e in enumerate(engines):
        for j, o in enumerate(engines):
            if i != j:
                blocks[j][e.row0:e.row1].copy_(blocks[i][e.row0:e.row1])
    torch.cuda.synchronize()


def lockstep_solve(engines, opts):
    for e in engines:
        e.begin(opts)
    for e in engines:
        e.phase(PH_SETUP_LOCAL, 0)
    exchange(engines, BLOCK_R, 0)
    for e in engines:
        e.phase(PH_SETUP_REST, 0)
    if opts.algo == "mccg":
        for e in engines:
            e.phase(PH_MCCG_SETUP, 0)
    stop = engines[0].state()[0]
    k = 0
    while True:
        while not stop and k < engines[0].max_iters:
            for e in engines:
                e.phase(PH_ITER_LOCAL, k)
            exchange(engines, BLOCK_Q, k)
            for e in engines:
                e.phase(PH_ITER_MID, k)
            if engines[0].recompute_at(k):
                exchange(engines, BLOCK_R, k)
            for e in engines:
                e.phase(PH_ITER_REST, k)
            k += 1
            stops = [e.state()[0] for e in engines]
            assert len(set(stops)) == 1  # replicated state => identical decisions
            stop = stops[0]
        if not (opts.algo == "mccg" and stop):
            break
        ks = [e.mccg_resume() for e in engines]  # every shard restricts identically
        assert len(set(ks)) == 1
        if ks[0] < 0:
            break
        k, stop = ks[0], False
    for e in engines:
        e.phase(PH_FINAL_LOCAL, 0)
    exchange(engines, BLOCK_S, 0)
    for e in engines:
        e.phase(PH_FINAL_REST, 0)
    return [e.end() for e in engines]


@pytest.mark.parametrize("n,p,world,max_iters", [(600, 4, 2, -1), (517, 8, 3, 60), (256, 16, 2, 55)])
def test_sharded_exact_bitwise(po, n, p, world, max_iters):
    import paper_1204_0069_b200 as m
    A = po.gen_diagdom(n, n) if p != 4 else po.gen_householder(n, 8, 1e3, n)
    b = po.gen_rhs(n, "uniform", n)
    X0 = po.gen_starts(n, p, n)
    opts = m.SolveOptions(tol=(1e-10 * po.seq_norm(b) if max_iters < 0 else 0.0), max_iters=max_iters)
    engines = [GpuShardEngine(n, p, r, world, 0, "exact") for r in range(world)]
    for e in engines:
        e.ctx.set_A(A[e.row0:e.row1])
        e.ctx.upload(b, X0)
    traces = lockstep_solve(engines, opts)
    ref = po.oracle_ccg(A, b, X0, tol=opts.tol, max_iters=max_iters)
    for t in traces:
        assert str(t.status) == ref.status and t.iteration_count() == ref.iterations
        assert np.array_equal(t.residual_norms, ref.residual_norms)
        assert np.array_equal(t.final_x, ref.final_x)
        assert np.array_equal(t.final_residual_norms, ref.final_residual_norms)
    for e in engines:
        e.close()


def test_sharded_generated_diagdom_matches_single(po):
    """Shards generate their own rows of A on the device (gen_A on a shard)."""
    import paper_1204_0069_b200 as m
    n, p, world = 700, 8, 2
    engines = [GpuShardEngine(n, p, r, world, 0, "exact") for r in range(world)]
    b = m.gen_rhs(n, "uniform", 3)
    X0 = m.gen_starts(n, p, 3)
    for e in engines:
        e.ctx.gen_A("diagdom", 3)
        assert np.array_equal(e.ctx.get_A(), po.gen_diagdom(n, 3)[e.row0:e.row1])
        e.ctx.upload(b, X0)
    opts = m.SolveOptions(max_iters=40)
    traces = lockstep_solve(engines, opts)
    with m.GpuContext(n, p) as ctx:
        ctx.gen_A("diagdom", 3)
        single = ctx.solve(b, X0, opts)
    assert np.array_equal(traces[0].final_x, single.final_x)
    assert np.array_equal(traces[1].residual_norms, single.residual_norms)
    for e in engines:
        e.close()


def test_sharded_fast_within_tolerance(po):
    import paper_1204_0069_b200 as m
    n, p, world = 900, 8, 2
    A = po.gen_diagdom(n, 11)
    b = po.gen_rhs(n, "uniform", 11)
    X0 = po.gen_starts(n, p, 11)
    opts = m.SolveOptions(tol=1e-10 * po.seq_norm(b))
    engines = [GpuShardEngine(n, p, r, world, 0, "fast") for r in range(world)]
    for e in engines:
        e.ctx.set_A(A[e.row0:e.row1])
        e.ctx.upload(b, X0)
    traces = lockstep_solve(engines, opts)
    ref = po.oracle_ccg(A, b, X0, tol=opts.tol)
    for t in traces:
        assert str(t.status) == "converged" and abs(t.iteration_count() - ref.iterations) <= 2
        rel = np.linalg.norm(t.final_x - ref.final_x, axis=0) / np.linalg.norm(ref.final_x, axis=0)
        assert rel.max() < 1e-8
    assert np.array_equal(traces[0].final_x, traces[1].final_x)  # ranks agree bit for bit
    for e in engines:
        e.close()


@pytest.mark.parametrize("n,world", [(257, 2), (385, 2), (386, 3)])
def test_sharded_fast_long_run_on_unequal_shards(po, n, world):
    """The phase API on UNEQUAL row shards (129 + 128 rows, 193 + 192, 129 + 129 +
    128: the old row-pass grids differed between the ranks) for a long fast-mode
    solve: every rank must hold the same replicated X, R, D bit for bit at the end
    -- the Gram row pass groups its partial sums by n, not by the shard's own row
    count (tests/test_gpu_multi.py, profiles/r02_fuzz_parity.txt)."""
    import paper_1204_0069_b200 as m
    p, seed = 4, 1600630417
    A = po.gen_householder(n, 3, 3.3e3, seed)
    b = po.gen_rhs(n, "normal", seed)
    X0 = po.gen_starts(n, p, seed)
    opts = m.SolveOptions(tol=2.4e-10 * po.seq_norm(b))
    engines = [GpuShardEngine(n, p, r, world, 0, "fast") for r in range(world)]
    assert len({e.row1 - e.row0 for e in engines}) > 1  # unequal shards
    for e in engines:
        e.ctx.set_A(A[e.row0:e.row1])
        e.ctx.upload(b, X0)
    traces = lockstep_solve(engines, opts)
    ref = po.oracle_ccg(A, b, X0, tol=opts.tol)
    assert ref.status == "converged" and ref.iterations > 60
    for t in traces:
        assert str(t.status) == "converged" and abs(t.iteration_count() - ref.iterations) <= max(4, ref.iterations // 20)
        assert np.array_equal(t.final_x, traces[0].final_x)          # ranks agree bit for bit
        assert np.array_equal(t.residual_norms, traces[0].residual_norms)
    rel = np.linalg.norm(traces[0].final_x - ref.final_x, axis=0) / np.linalg.norm(ref.final_x, axis=0)
    assert rel.max() < 10 * 3.3e3 * 2.4e-10
    for e in engines:
        e.close()


@pytest.mark.parametrize("name,world", [("mccg_n50_p8", 2), ("mccg_exhaustion_cliff", 3),
                                        ("mccg_duplicate_columns", 2)])
def test_sharded_mccg_matches_reference(name, world):
    """mccg_solve on row-sharded contexts: each shard restricts its replicated
    blocks on a rank drop (coopcg_gpu_mccg_resume) and the trace equals the
    reference's own (golden fixture), NaN rows for dropped agents included."""
    import paper_1204_0069_b200 as m
    from conftest import load_golden
    A, z = load_golden(name)
    n, p = z["X0"].shape
    opts = m.SolveOptions(tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                          recompute_residual_every=int(z["recompute"]), algo="mccg")
    engines = [GpuShardEngine(n, p, r, world, 0, "exact") for r in range(world)]
    for e in engines:
        e.ctx.set_A(A[e.row0:e.row1])
        e.ctx.upload(z["b"], z["X0"])
    traces = lockstep_solve(engines, opts)
    act = [int(a) for a in z["active_agents"]]
    for t in traces:
        assert str(t.status) == str(z["status"]) and t.iteration_count() == int(z["iterations"])
        assert t.converged_agent == int(z["converged_agent"])
        assert np.array_equal(t.residual_norms, z["residual_norms"], equal_nan=True)
        assert t.active_agents == act
        assert np.array_equal(t.final_x, z["final_x"][:, act])
        assert np.array_equal(t.final_residual_norms_by_id, z["final_residual_norms"], equal_nan=True)
    for e in engines:
        e.close()


class _LockstepW:
    """In-process stand-in for the n x 1 all-gather of w between shards."""

    def __init__(self, engines):
        self.engines = engines

    def run(self, seed, m, kappa):
        from paper_1204_0069_b200 import _capi
        from paper_1204_0069_b200.sharded import BLOCK_W
        from paper_1204_0069_b200.solver import _check
        L = _capi.lib()
        for e in self.engines:
            _check(e.ctx._h, L.coopcg_gpu_gen_householder_begin(e.ctx._h, seed, m, kappa))
        ws = [e.vector(BLOCK_W) for e in self.engines]
        for r in range(m - 1, -1, -1):
            for e in self.engines:
                _check(e.ctx._h, L.coopcg_gpu_gen_householder_local(e.ctx._h, r))
            torch.cuda.synchronize()
            for i, e in enumerate(self.engines):
                for j in range(len(self.engines)):
                    if i != j:
                        ws[j][e.row0:e.row1].copy_(ws[i][e.row0:e.row1])
            torch.cuda.synchronize()
            for e in self.engines:
                _check(e.ctx._h, L.coopcg_gpu_gen_householder_rest(e.ctx._h, r))
        for e in self.engines:
            _check(e.ctx._h, L.coopcg_gpu_gen_householder_end(e.ctx._h))


@pytest.mark.parametrize("n,p,world,arith", [(517, 4, 3, "exact"), (256, 8, 2, "fast")])
def test_sharded_householder_generation(po, n, p, world, arith):
    """Row-sharded Householder generation (w all-gathered per reflector): every
    shard's rows equal the oracle's full matrix bit for bit, and the sharded
    solve on them equals the oracle solve (exact)."""
    import paper_1204_0069_b200 as m
    seed, refl, kappa = 11, 6, 1e3
    A = po.gen_householder(n, refl, kappa, seed)
    engines = [GpuShardEngine(n, p, r, world, 0, arith) for r in range(world)]
    _LockstepW(engines).run(seed, refl, kappa)
    for e in engines:
        assert np.array_equal(e.ctx.get_A(), A[e.row0:e.row1])
    if arith == "exact":
        b = po.gen_rhs(n, "normal", seed)
        X0 = po.gen_starts(n, p, seed)
        opts = m.SolveOptions(tol=0.0, max_iters=40)
        for e in engines:
            e.ctx.upload(b, X0)
        traces = lockstep_solve(engines, opts)
        ot = po.oracle_ccg(A, b, X0, tol=0.0, max_iters=40)
        for t in traces:
            assert np.array_equal(t.residual_norms, ot.residual_norms)
            assert np.array_equal(t.final_x, ot.final_x)
    for e in engines:
        e.close()
