"""ctypes binding to the oracle libraries.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg import this module, and only as the checker or the
timed CPU baseline -- never as part of the product path.

Two libraries:
  * ``oracle/_build/liboracle.so`` -- the plain-C restatement of the reference
    solver and of the BASELINE generators (ccg_oracle.c, gen_oracle.c);
  * ``oracle/_ref/libccgref.so``   -- the reference headers themselves, compiled
    by ``oracle/Makefile`` (``make ref``) in the container that has
    /root/reference; the built .so travels to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libccgref.so")

STATUS_NAMES = {0: "converged", 1: "rank-collapse", 2: "max-iterations"}


class OrcOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int),
                ("recompute_residual_every", C.c_int), ("rank_rel_tol", C.c_double)]


class OrcTrace(C.Structure):
    _fields_ = [("status", C.c_int), ("converged_agent", C.c_int), ("iterations", C.c_int),
                ("capacity", C.c_int),
                ("residual_norms", C.POINTER(C.c_double)), ("minres", C.POINTER(C.c_double)),
                ("wall_ns", C.POINTER(C.c_uint64)),
                ("initial_residual_norms", C.POINTER(C.c_double)), ("initial_minres", C.c_double),
                ("final_x", C.POINTER(C.c_double)),
                ("final_residual_norms", C.POINTER(C.c_double)), ("final_minres", C.c_double),
                ("loop_wall_ns", C.c_uint64), ("error_msg", C.c_char * 256),
                ("active_agents", C.POINTER(C.c_int)), ("n_active", C.c_int)]


@dataclass
class Trace:
    rc: int
    error: str
    status: str
    converged_agent: int
    iterations: int
    residual_norms: np.ndarray  # (iterations, p)
    minres: np.ndarray
    wall_ns: np.ndarray
    initial_residual_norms: np.ndarray
    initial_minres: float
    final_x: np.ndarray  # (n, p)
    final_residual_norms: np.ndarray
    final_minres: float
    loop_wall_ns: int
    extra: dict = field(default_factory=dict)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


_libs: dict = {}


def oracle_lib() -> C.CDLL:
    if "orc" not in _libs:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_SO)
        lib.orc_ccg_solve.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(OrcOpts), C.POINTER(OrcTrace)]
        lib.orc_mccg_solve.argtypes = lib.orc_ccg_solve.argtypes
        lib.orc_dot.restype = C.c_double
        lib.orc_dot.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
        lib.orc_gen_diagdom.argtypes = [C.c_int, C.c_uint64, C.c_void_p]
        lib.orc_gen_householder_factors.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64,
                                                    C.c_void_p, C.c_void_p]
        lib.orc_gen_householder.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.orc_gen_rhs.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        lib.orc_gen_starts.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        lib.orc_numerical_rank.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]
        lib.orc_solve_small.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        lib.orc_gram.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        lib.orc_matvec_block.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        lib.orc_gen_diagdom_rows.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        lib.orc_gen_householder_par.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _libs["orc"] = lib
    return _libs["orc"]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib(path: str = REF_SO) -> C.CDLL:
    """The compiled reference (path: another build of the same shim, e.g. the
    FMA-contracted twin oracle/_ref/libccgref_fma.so of tests/golden/make_kdiv.py)."""
    key = "ref" if path == REF_SO else path
    if key not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(path)
        lib.ref_block_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(OrcOpts), C.POINTER(OrcTrace)]
        lib.ref_cg_solve.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(OrcOpts), C.POINTER(OrcTrace)]
        lib.ref_sd_solve.argtypes = lib.ref_cg_solve.argtypes
        lib.ref_make_problem.argtypes = [C.c_int, C.c_int, C.c_double, C.c_ulonglong,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_random_spd.argtypes = [C.c_int, C.c_double, C.c_ulonglong, C.c_void_p, C.c_void_p]
        lib.ref_matvec_block.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_gram.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_solve_small.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        lib.ref_numerical_rank.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_void_p]
        lib.ref_matrix_new.restype = C.c_void_p
        lib.ref_matrix_new.argtypes = [C.c_int]
        lib.ref_matrix_data.restype = C.POINTER(C.c_double)
        lib.ref_matrix_data.argtypes = [C.c_void_p]
        lib.ref_matrix_free.argtypes = [C.c_void_p]
        lib.ref_block_solve_m.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                          C.POINTER(OrcOpts), C.POINTER(OrcTrace)]
        _libs[key] = lib
    return _libs[key]


def _run(fn, n, p, capacity, *args) -> Trace:
    norms = np.full((max(capacity, 1), p), np.nan)
    minres = np.zeros(max(capacity, 1))
    wall = np.zeros(max(capacity, 1), dtype=np.uint64)
    init = np.zeros(p)
    fx = np.zeros((p, n))  # column-major n x p == row-major p x n
    fr = np.zeros(p)
    act = np.zeros(p, dtype=np.int32)
    tr = OrcTrace()
    tr.active_agents = act.ctypes.data_as(C.POINTER(C.c_int))
    tr.capacity = capacity
    tr.residual_norms = _dp(norms)
    tr.minres = _dp(minres)
    tr.wall_ns = wall.ctypes.data_as(C.POINTER(C.c_uint64))
    tr.initial_residual_norms = _dp(init)
    tr.final_x = _dp(fx)
    tr.final_residual_norms = _dp(fr)
    rc = fn(*args, C.byref(tr))
    it = min(tr.iterations, capacity)
    return Trace(rc=rc, error=tr.error_msg.decode(), status=STATUS_NAMES.get(tr.status, "?"),
                 converged_agent=tr.converged_agent, iterations=tr.iterations,
                 residual_norms=norms[:it].copy(), minres=minres[:it].copy(), wall_ns=wall[:it].copy(),
                 initial_residual_norms=init, initial_minres=tr.initial_minres,
                 final_x=fx.T.copy(), final_residual_norms=fr, final_minres=tr.final_minres,
                 loop_wall_ns=int(tr.loop_wall_ns),
                 extra={"active_agents": act[:tr.n_active].tolist()})


def _opts(tol, max_iters, recompute, rank_tol):
    o = OrcOpts()
    o.tol = tol
    o.max_iters = max_iters
    o.recompute_residual_every = recompute
    o.rank_rel_tol = rank_tol
    return o


def _prep(A, b, X0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    X0 = np.asarray(X0, dtype=np.float64)
    n, p = X0.shape
    X0c = np.ascontiguousarray(X0.T)  # column-major
    return A, b, X0c, n, p


def oracle_ccg(A, b, X0, tol=0.0, max_iters=-1, recompute=-1, rank_tol=1e-10, algo="ccg") -> Trace:
    """The C restatement of ccg_solve (algo="mccg": mccg_solve).  X0 is an (n, p) array."""
    A, b, X0c, n, p = _prep(A, b, X0)
    cap = max_iters if max_iters >= 0 else 2 * n
    o = _opts(tol, max_iters, recompute, rank_tol)
    fn = oracle_lib().orc_ccg_solve if algo == "ccg" else oracle_lib().orc_mccg_solve
    return _run(fn, n, p, cap, n, p, A.ctypes.data, b.ctypes.data, X0c.ctypes.data, C.byref(o))


def ref_solve(A, b, X0, tol=0.0, max_iters=-1, recompute=-1, rank_tol=1e-10, algo="ccg") -> Trace:
    """The reference itself: algo in {"ccg", "parallel", "mccg"}."""
    A, b, X0c, n, p = _prep(A, b, X0)
    cap = max_iters if max_iters >= 0 else 2 * n
    o = _opts(tol, max_iters, recompute, rank_tol)
    code = {"ccg": 0, "parallel": 1, "mccg": 2, "parallel_team_finalize": 3}[algo]
    return _run(ref_lib().ref_block_solve, n, p, cap, code, n, p, A.ctypes.data, b.ctypes.data,
                X0c.ctypes.data, C.byref(o))


class RefMatrix:
    """An n x n system matrix owned by the reference shim (one host copy: the
    entries are written in place, then moved into the reference's SpdMatrix).
    For the full-size BASELINE configs, where A is 2-137 GB."""

    def __init__(self, n: int, lib_path: str = REF_SO):
        self.n = n
        self._lib = ref_lib(lib_path)
        self._h = self._lib.ref_matrix_new(n)
        if not self._h:
            raise MemoryError(f"ref_matrix_new({n}) failed ({8 * n * n / 1e9:.1f} GB)")
        ptr = self._lib.ref_matrix_data(self._h)
        self.A = np.ctypeslib.as_array(ptr, shape=(n, n))  # writable view of the entries

    def solve(self, b, X0, tol=0.0, max_iters=-1, recompute=-1, rank_tol=1e-10, algo="parallel") -> Trace:
        b = np.ascontiguousarray(b, dtype=np.float64)
        X0 = np.asarray(X0, dtype=np.float64)
        n, p = X0.shape
        assert n == self.n
        X0c = np.ascontiguousarray(X0.T)
        cap = max_iters if max_iters >= 0 else 2 * n
        o = _opts(tol, max_iters, recompute, rank_tol)
        code = {"ccg": 0, "parallel": 1, "mccg": 2, "parallel_team_finalize": 3}[algo]
        return _run(self._lib.ref_block_solve_m, n, p, cap, code, self._h, p, b.ctypes.data,
                    X0c.ctypes.data, C.byref(o))

    def close(self):
        if self._h:
            self.A = None
            self._lib.ref_matrix_free(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def ref_cg(A, b, x0, tol=0.0, max_iters=-1, recompute=-1, algo="cg") -> Trace:
    """The reference's cg_solve (algo="sd": steepest_descent_solve)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    n = len(b)
    cap = max_iters if max_iters >= 0 else 2 * n
    o = _opts(tol, max_iters, recompute, 1e-10)
    fn = ref_lib().ref_cg_solve if algo == "cg" else ref_lib().ref_sd_solve
    return _run(fn, n, 1, cap, n, A.ctypes.data, b.ctypes.data, x0.ctypes.data, C.byref(o))


def ref_random_spd(n, cond, seed):
    """The reference's random_spd_with_spectrum: (A row-major, spectrum)."""
    A = np.zeros((n, n))
    lam = np.zeros(n)
    if ref_lib().ref_random_spd(n, cond, seed, A.ctypes.data, lam.ctypes.data) != 0:
        raise RuntimeError("ref_random_spd failed")
    return A, lam


def ref_make_problem(n, p, cond, seed):
    A = np.zeros((n, n))
    b = np.zeros(n)
    X0c = np.zeros((p, n))
    rc = ref_lib().ref_make_problem(n, p, cond, seed, A.ctypes.data, b.ctypes.data, X0c.ctypes.data)
    if rc != 0:
        raise RuntimeError("ref_make_problem failed")
    return A, b, X0c.T.copy()


# ---- BASELINE generators (restatement) -------------------------

def gen_diagdom(n, seed):
    A = np.zeros((n, n))
    oracle_lib().orc_gen_diagdom(n, seed, A.ctypes.data)
    return A


def gen_diagdom_rows(n, seed, r0, r1, out=None):
    """Rows [r0, r1) of gen_diagdom(n, seed) (OpenMP over rows, same bits)."""
    if out is None:
        out = np.empty((r1 - r0, n))
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == (r1 - r0) * n
    oracle_lib().orc_gen_diagdom_rows(n, seed, r0, r1, out.ctypes.data)
    return out


def gen_householder_into(n, m, kappa, seed, out):
    """gen_householder(n, m, kappa, seed) written into `out` (OpenMP over rows, same bits)."""
    V, lam = gen_householder_factors(n, m, kappa, seed)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == n * n
    oracle_lib().orc_gen_householder_par(n, m, V.ctypes.data, lam.ctypes.data, out.ctypes.data)
    return out


def gen_householder_factors(n, m, kappa, seed):
    V = np.zeros((m, n))
    lam = np.zeros(n)
    oracle_lib().orc_gen_householder_factors(n, m, kappa, seed, V.ctypes.data, lam.ctypes.data)
    return V, lam


def gen_householder(n, m, kappa, seed):
    V, lam = gen_householder_factors(n, m, kappa, seed)
    A = np.zeros((n, n))
    oracle_lib().orc_gen_householder(n, m, V.ctypes.data, lam.ctypes.data, A.ctypes.data)
    return A


def gen_rhs(n, kind, seed):
    b = np.zeros(n)
    oracle_lib().orc_gen_rhs(n, 0 if kind == "uniform" else 1, seed, b.ctypes.data)
    return b


def gen_starts(n, p, seed):
    X0c = np.zeros((p, n))
    oracle_lib().orc_gen_starts(n, p, seed, X0c.ctypes.data)
    return X0c.T.copy()


def seq_norm(b) -> float:
    """sqrt(dot(b, b)) in ascending order (the tolerance scale)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(np.sqrt(oracle_lib().orc_dot(b.ctypes.data, b.ctypes.data, len(b))))


def numerical_rank(D, tol, lib="oracle"):
    D = np.asarray(D, dtype=np.float64)
    n, p = D.shape
    Dc = np.ascontiguousarray(D.T)
    cols = np.zeros(p, dtype=np.int32)
    if lib == "oracle":
        r = oracle_lib().orc_numerical_rank(Dc.ctypes.data, n, p, tol, cols.ctypes.data)
    else:
        r = ref_lib().ref_numerical_rank(n, p, Dc.ctypes.data, tol, cols.ctypes.data)
    return r, cols[:r].copy()
