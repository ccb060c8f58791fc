"""The oracle (plain-C restatement of ccg_solve) is pinned against the
reference: the golden fixtures the reference produced (tests/golden/, made by
make_golden.py from oracle/_ref) and, where the reference shim is built, a
direct bit-for-bit comparison on fresh seeded inputs."""
import hashlib

import numpy as np
import pytest

from conftest import golden_names, load_golden


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def assert_trace_equal(t, z):
    assert t.rc == int(z["rc"])
    if t.rc != 0:
        return
    if "active_agents" in z and len(z["active_agents"]):
        assert t.extra["active_agents"] == [int(a) for a in z["active_agents"]]
    assert t.status == str(z["status"])
    assert t.iterations == int(z["iterations"])
    assert t.converged_agent == int(z["converged_agent"])
    # bitwise: per-iteration per-agent norms, minres, final X, true residuals
    assert np.array_equal(t.residual_norms, z["residual_norms"], equal_nan=True)
    assert np.array_equal(t.minres, z["minres"])
    assert np.array_equal(t.initial_residual_norms, z["initial_residual_norms"])
    assert np.array_equal(t.final_x, z["final_x"], equal_nan=True)
    assert np.array_equal(t.final_residual_norms, z["final_residual_norms"], equal_nan=True)
    assert t.final_minres == float(z["final_minres"])


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_golden(po, name):
    A, z = load_golden(name)
    assert _sha(A) == str(z["A_sha256"]), "generator drifted from the pinned bytes"
    algo = str(z["algo"]) if "algo" in z else "ccg"
    if algo == "sd":
        pytest.skip("steepest descent: pinned by the GPU test against the reference fixture directly")
    rec = int(z["recompute"])
    if algo == "cg":  # cg_solve == the p = 1 block solver, recompute default 1 (test_solvers.cpp:176-201)
        algo, rec = "ccg", (1 if rec < 0 else rec)
    t = po.oracle_ccg(A, z["b"], z["X0"], tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                      recompute=rec, algo=algo)
    assert_trace_equal(t, z)


@pytest.mark.skipif(not __import__("pyoracle").ref_available(), reason="reference shim not built")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_reference_live(po, seed):
    rng = np.random.default_rng(seed)
    n, p = int(rng.integers(40, 160)), int(rng.integers(1, 7))
    A, b, X0 = po.ref_make_problem(n, p, float(10 ** rng.uniform(1, 4)), seed)
    a = po.oracle_ccg(A, b, X0, tol=1e-9)
    r = po.ref_solve(A, b, X0, tol=1e-9)
    assert a.status == r.status and a.iterations == r.iterations
    assert np.array_equal(a.residual_norms, r.residual_norms)
    assert np.array_equal(a.final_x, r.final_x)
    pr = po.ref_solve(A, b, X0, tol=1e-9, algo="parallel")  # parallel_ccg == ccg_solve bitwise
    assert np.array_equal(pr.final_x, r.final_x) and np.array_equal(pr.residual_norms, r.residual_norms)


def _trace_fields_equal(a, b):
    assert a.rc == b.rc and a.status == b.status and a.iterations == b.iterations
    assert a.converged_agent == b.converged_agent
    for f in ("initial_residual_norms", "residual_norms", "minres", "final_x", "final_residual_norms"):
        assert np.array_equal(getattr(a, f), getattr(b, f), equal_nan=True), f
    assert a.final_minres == b.final_minres or (np.isnan(a.final_minres) and np.isnan(b.final_minres))


@pytest.mark.skipif(not __import__("pyoracle").ref_available(), reason="reference shim not built")
@pytest.mark.parametrize("case", ["converged", "fixed", "degenerate", "rank_loop", "recompute"])
def test_team_finalize_equals_parallel_ccg(po, case):
    """The full-size parity test's reference at cfg 3 / 4 (ref_shim.cpp,
    parallel_ccg_team_finalize: finalize_trace's agent loop run by the team)
    gives parallel_ccg's trace bit for bit."""
    n, p = 300, 5
    # rank_loop: three distinct eigenvalues, so D loses rank inside the loop (k = 20)
    A = po.gen_diagdom(n, 7) if case != "rank_loop" else np.diag(np.repeat([1.0, 2.0, 5.0], n // 3))
    b = po.gen_rhs(n, "uniform", 7)
    X0 = po.gen_starts(n, p, 7)
    kw = dict(tol=1e-10 * po.seq_norm(b), max_iters=-1)
    if case == "fixed":
        kw = dict(tol=0.0, max_iters=25)
    elif case == "degenerate":
        X0 = np.zeros((n, p))
    elif case == "rank_loop":
        kw = dict(tol=0.0, max_iters=50)
    elif case == "recompute":
        kw = dict(tol=0.0, max_iters=30, recompute=7)
    a = po.ref_solve(A, b, X0, algo="parallel", **kw)
    t = po.ref_solve(A, b, X0, algo="parallel_team_finalize", **kw)
    _trace_fields_equal(a, t)


@pytest.mark.skipif(not __import__("pyoracle").ref_available(), reason="reference shim not built")
def test_oracle_kernels_match_reference(po):
    import ctypes as C
    rng = np.random.default_rng(5)
    n, p = 70, 5
    A, _, _ = po.ref_make_problem(n, p, 100.0, 9)
    D = rng.uniform(-1, 1, (n, p))
    Dc = np.ascontiguousarray(D.T)
    o1 = np.zeros((p, n))
    o2 = np.zeros((p, n))
    po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, o1.ctypes.data)
    po.ref_lib().ref_matvec_block(n, p, A.ctypes.data, Dc.ctypes.data, o2.ctypes.data)
    assert np.array_equal(o1, o2)
    # numerical_rank: full, (v, 2v, w), zero block (tests/test_dense.cpp:246-291)
    for blk in (D, np.stack([D[:, 0], 2 * D[:, 0], D[:, 1]], 1), np.zeros((n, 3))):
        assert po.numerical_rank(blk, 1e-10) [0] == po.numerical_rank(blk, 1e-10, lib="ref")[0]


def test_generators_are_symmetric_and_spd(po):
    A = po.gen_diagdom(64, 3)
    assert np.array_equal(A, A.T)
    assert np.all(np.diag(A) > np.sum(np.abs(A), 1) - np.diag(A))
    H = po.gen_householder(48, 4, 1e3, 3)
    assert np.array_equal(H, H.T)
    ev = np.linalg.eigvalsh(H)
    assert ev.min() > 0.5 and ev.max() < 1.1e3


def test_degenerate_x0_rank_collapse(po):
    A = po.gen_diagdom(100, 1)
    b = po.gen_rhs(100, "uniform", 1)
    t = po.oracle_ccg(A, b, np.zeros((100, 3)), tol=1e-10)
    assert t.status == "rank-collapse" and t.iterations == 0
