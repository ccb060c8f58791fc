"""Host-side mirror of the reference solver API over the CUDA C ABI.

Reference interface mirrored (names, argument meaning, error behaviour):
  * ``ccg_solve(A, b, X0, opts)``      coopcg/solvers.hpp:329-333
  * ``SolveOptions``                   coopcg/trace.hpp:74-88
  * ``SolveTrace`` / ``IterationRecord`` coopcg/trace.hpp:33-71
  * ``TerminalStatus``                 coopcg/trace.hpp:13-29
  * exceptions                         coopcg/errors.hpp:11-41
  * mult counting convention           coopcg/workplan.hpp:26-59

Everything numeric runs in the CUDA library (``_capi``); this module only
marshals host buffers.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi


# ---- errors (errors.hpp:11-41) ------------------------------------------------
class Error(RuntimeError):
    """Base class for all library errors (errors.hpp:15-18)."""


class DimensionError(Error):
    pass


class SingularMatrixError(Error):
    pass


class SpdViolationError(Error):
    pass


class NumericalBreakdownError(Error):
    pass


class CudaError(Error):
    pass


_ERRORS = {1: DimensionError, 2: SpdViolationError, 3: NumericalBreakdownError,
           4: SingularMatrixError, 5: Error, 6: Error, 10: CudaError}


class TerminalStatus(enum.IntEnum):
    Converged = 0
    RankCollapse = 1
    MaxIterations = 2

    def __str__(self) -> str:  # to_string (trace.hpp:19-29)
        return {0: "converged", 1: "rank-collapse", 2: "max-iterations"}[int(self)]


@dataclass
class SolveOptions:
    tol: float = 0.0
    max_iters: int = -1
    recompute_residual_every: int = -1
    rank_rel_tol: float = 1e-10
    algo: str = "ccg"  # "ccg" (ccg_solve) | "mccg" (mccg_solve, solvers.hpp:338-342) | "sd" (internal)
    # verification mode (trace.hpp:86-87): retain X_k, R_k, D_k; record A-norm errors against x_star
    keep_history: bool = False
    x_star: Optional[np.ndarray] = None

    def to_c(self) -> _capi.coopcg_opts:
        o = _capi.coopcg_opts()
        o.tol = float(self.tol)
        o.max_iters = int(self.max_iters)
        o.recompute_residual_every = int(self.recompute_residual_every)
        o.rank_rel_tol = float(self.rank_rel_tol)
        o.algo = {"ccg": 0, "mccg": 1, "sd": 2}[self.algo]
        return o


@dataclass
class GpuOptions:
    device: int = 0
    arith: str = "exact"  # "exact" (bit-identical to the reference) | "fast"
    # several devices: A row-block sharded over them, one process driving all
    # (coopcg_gpu_create_multi; a device may repeat).  None: `device` alone.
    devices: Optional[List[int]] = None


@dataclass
class IterationRecord:
    k: int
    active_agents: int
    agents: List[int]
    residual_norms: np.ndarray
    minres: float
    mults: int
    mults_per_worker: List[int]
    wall_ns: int
    anorm_errors: Optional[np.ndarray] = None  # per agent ||x_j - x*||_A when SolveOptions.x_star is set


@dataclass
class SolveTrace:
    iterations: List[IterationRecord]
    status: TerminalStatus
    converged_agent: int
    final_x: np.ndarray  # (n, p)
    active_agents: List[int]
    initial_residual_norms: np.ndarray
    initial_minres: float
    final_residual_norms: np.ndarray
    final_minres: float
    setup_mults: int
    loop_wall_ns: int
    final_residual_norms_by_id: np.ndarray = field(default=None)
    barriers_per_iteration: int = 0
    residual_norms: np.ndarray = field(default=None)  # (iterations, p)
    minres: np.ndarray = field(default=None)
    wall_ns: np.ndarray = field(default=None)
    exact_rank_checks: int = 0
    # keep_history: entry 0 is the initial block, entry k + 1 the state after iteration k (trace.hpp:66-70)
    history_x: List[np.ndarray] = field(default_factory=list)
    history_r: List[np.ndarray] = field(default_factory=list)
    history_d: List[np.ndarray] = field(default_factory=list)

    def iteration_count(self) -> int:
        return len(self.iterations)


def _lu_mults(p: int) -> int:
    return p * (p + 1) * (2 * p + 1) // 6


def iteration_mults(n: int, p: int, recompute: bool) -> int:
    """Per-worker counted multiplications of one iteration (workplan.hpp:693-715)."""
    resid = n * n if recompute else n * p
    return n * n + 5 * n * p + resid + 2 * _lu_mults(p)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(ctx_handle, rc: int) -> None:
    if rc == 0:
        return
    buf = C.create_string_buffer(512)
    _capi.lib().coopcg_gpu_last_error(ctx_handle, buf, 512)  # None: the thread's last create/host error
    msg = buf.value.decode() or f"coopcg error code {rc}"
    raise _ERRORS.get(rc, Error)(msg)


_ARITH = {"exact": 0, "fast": 1}


class GpuContext:
    """One solver context on one GPU (owns device memory and a CUDA stream).

    ``row_begin``/``row_end`` select a row block of A for sharded multi-GPU
    solves (see ``paper_1204_0069_b200.sharded``); the default is the whole
    matrix.
    """

    def __init__(self, n: int, p: int, device: int = 0, arith: str = "exact",
                 row_begin: int = 0, row_end: Optional[int] = None, devices: Optional[List[int]] = None,
                 nccl: Optional[tuple] = None):
        """devices: row-shard A over these devices, one process driving all
        (coopcg_gpu_create_multi).  nccl = (nranks, rank, unique_id_bytes):
        this process's rank context (coopcg_gpu_create_rank) with the NCCL row
        exchanges inside the library; its rows are row_split(n, nranks, rank)."""
        L = _capi.lib()
        self.n, self.p, self.device, self.arith = n, p, device, arith
        self.devices = list(devices) if devices else [device]
        self.row_begin = row_begin
        self.row_end = n if row_end is None else row_end
        h = C.c_void_p()
        if arith not in _ARITH:
            raise Error(f"unknown arith mode {arith!r}")
        if nccl is not None:
            nranks, rank, uid = nccl
            if len(uid) != _capi.NCCL_ID_BYTES:
                raise Error("nccl unique id must be 128 bytes (nccl_unique_id())")
            self.row_begin, self.row_end = row_split(n, nranks, rank)
            idbuf = C.create_string_buffer(bytes(uid), _capi.NCCL_ID_BYTES)
            rc = L.coopcg_gpu_create_rank(n, p, device, _ARITH[arith], nranks, rank, idbuf, C.byref(h))
        elif devices is not None and len(devices) > 1:
            arr = (C.c_int * len(devices))(*devices)
            rc = L.coopcg_gpu_create_multi(n, p, len(devices), arr, _ARITH[arith], C.byref(h))
        else:
            rc = L.coopcg_gpu_create_shard(n, p, device, _ARITH[arith], self.row_begin, self.row_end,
                                           C.byref(h))
        if rc != 0:
            buf = C.create_string_buffer(512)
            L.coopcg_gpu_last_error(None, buf, 512)
            raise _ERRORS.get(rc, Error)(buf.value.decode() or f"create failed ({rc})")
        self._h = h
        self._timing = _capi.coopcg_timing()

    def shards(self) -> list:
        """[(device, row_begin, row_end)] of the context's row shards."""
        ns = C.c_int()
        cap = 16
        dev, r0, r1 = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
        _check(self._h, _capi.lib().coopcg_gpu_shards(self._h, cap, C.byref(ns), dev, r0, r1))
        return [(dev[g], r0[g], r1[g]) for g in range(min(ns.value, cap))]

    # -- lifecycle --
    def close(self) -> None:
        if getattr(self, "_h", None):
            _capi.lib().coopcg_gpu_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the matrix --
    def set_A(self, A_rows: np.ndarray) -> None:
        A_rows = np.ascontiguousarray(A_rows, dtype=np.float64)
        if A_rows.shape != (self.row_end - self.row_begin, self.n):
            raise DimensionError("SpdMatrix: entry grid does not match dimension")
        _check(self._h, _capi.lib().coopcg_gpu_set_A(self._h, A_rows.ctypes.data))

    def gen_A(self, kind: str, seed: int, m: int = 0, kappa: float = 1.0) -> None:
        """Generate A on the device: "diagdom" / "householder" (the BASELINE
        generators) or "random_spd" (the reference's own
        random_spd(n, cond=kappa, seed), problem.hpp:118-152, bit-identical)."""
        k = {"diagdom": 0, "householder": 1, "random_spd": 2}[kind]
        _check(self._h, _capi.lib().coopcg_gpu_gen_A(self._h, k, seed, m, kappa))

    def get_A(self, row0: int = 0, rows: Optional[int] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Rows [row0, row0 + rows) of this context's row block (default: all)."""
        if rows is None:
            rows = self.row_end - self.row_begin - row0
        if out is None:
            out = np.empty((rows, self.n))
        elif out.dtype != np.float64 or not out.flags.c_contiguous or out.size != rows * self.n:
            raise DimensionError("get_A: output buffer does not match the row range")
        _check(self._h, _capi.lib().coopcg_gpu_get_A_rows(self._h, row0, rows, out.ctypes.data))
        return out

    # -- inputs / solve --
    def upload(self, b: np.ndarray, X0: np.ndarray) -> None:
        b = np.ascontiguousarray(b, dtype=np.float64)
        X0 = np.asarray(X0, dtype=np.float64)
        if b.shape != (self.n,) or X0.shape != (self.n, self.p):
            raise DimensionError("solver: operand shapes do not match the system matrix")
        X0c = np.ascontiguousarray(X0.T)  # DenseBlock column-major
        _check(self._h, _capi.lib().coopcg_gpu_upload(self._h, b.ctypes.data, X0c.ctypes.data))

    def run(self, opts: Optional[SolveOptions] = None, want_x: bool = True) -> SolveTrace:
        opts = opts or SolveOptions()
        n, p = self.n, self.p
        cap = max(opts.max_iters if opts.max_iters >= 0 else 2 * n, 1)
        norms = np.zeros((cap, p))
        minres = np.zeros(cap)
        wall = np.zeros(cap, dtype=np.uint64)
        init = np.zeros(p)
        fres = np.zeros(p)
        fx = np.zeros((p, n)) if want_x else None
        act = np.zeros(p, dtype=np.int32)
        tr = _capi.coopcg_trace()
        tr.active_agents = act.ctypes.data_as(C.POINTER(C.c_int))
        tr.capacity = cap
        tr.residual_norms = _dp(norms)
        tr.minres = _dp(minres)
        tr.wall_ns = wall.ctypes.data_as(C.POINTER(C.c_uint64))
        tr.initial_residual_norms = _dp(init)
        tr.final_residual_norms = _dp(fres)
        tr.final_x = _dp(fx) if want_x else C.POINTER(C.c_double)()
        co = opts.to_c()
        self._set_verification(opts)
        rc = _capi.lib().coopcg_gpu_run(self._h, C.byref(co), C.byref(tr))
        _check(self._h, rc)
        _capi.lib().coopcg_gpu_timing(self._h, C.byref(self._timing))
        t = self._make_trace(tr, norms, minres, wall, init, fres, fx, opts, act)
        self._read_verification(opts, t)
        return t

    def _set_verification(self, opts: SolveOptions) -> None:
        """SolveOptions.keep_history / x_star -> coopcg_gpu_set_verification (sticky per context)."""
        want = bool(opts.keep_history) or opts.x_star is not None
        if not want and not getattr(self, "_ver_on", False):
            return
        xs = None
        if opts.x_star is not None:
            xs = np.ascontiguousarray(opts.x_star, dtype=np.float64)
            if xs.shape != (self.n,):
                raise DimensionError("solver: operand shapes do not match the system matrix")
        _check(self._h, _capi.lib().coopcg_gpu_set_verification(
            self._h, 1 if opts.keep_history else 0, xs.ctypes.data if xs is not None else None))
        self._ver_on = want

    def _read_verification(self, opts: SolveOptions, t: "SolveTrace") -> None:
        L = _capi.lib()
        n, p, it = self.n, self.p, t.iteration_count()
        if opts.x_star is not None and it > 0:
            an = np.zeros((it, p))
            _check(self._h, L.coopcg_gpu_get_anorm_errors(self._h, it, an.ctypes.data))
            for rec in t.iterations:
                rec.anorm_errors = an[rec.k].copy()
        if opts.keep_history:
            cnt = C.c_int()
            _check(self._h, L.coopcg_gpu_history_count(self._h, C.byref(cnt)))
            for e in range(cnt.value):
                bufs = [np.zeros((p, n)) for _ in range(3)]
                _check(self._h, L.coopcg_gpu_get_history(self._h, e, *(b.ctypes.data for b in bufs)))
                t.history_x.append(bufs[0].T.copy())
                t.history_r.append(bufs[1].T.copy())
                t.history_d.append(bufs[2].T.copy())

    def run_raw(self, opts: Optional[SolveOptions] = None) -> tuple:
        """One solve through coopcg_gpu_run with reusable trace buffers and no
        Python trace assembly (the timed steps of bench.py).  Returns
        (iterations, exact_rank_checks); `run` is the full-trace API."""
        opts = opts or SolveOptions()
        cap = max(opts.max_iters if opts.max_iters >= 0 else 2 * self.n, 1)
        key = (cap, self.p)
        if getattr(self, "_raw", None) is None or self._raw[0] != key:
            bufs = [np.zeros((cap, self.p)), np.zeros(cap), np.zeros(cap, dtype=np.uint64), np.zeros(self.p),
                    np.zeros(self.p), np.zeros(self.p, dtype=np.int32)]
            tr = _capi.coopcg_trace()
            tr.capacity = cap
            tr.residual_norms = _dp(bufs[0])
            tr.minres = _dp(bufs[1])
            tr.wall_ns = bufs[2].ctypes.data_as(C.POINTER(C.c_uint64))
            tr.initial_residual_norms = _dp(bufs[3])
            tr.final_residual_norms = _dp(bufs[4])
            tr.active_agents = bufs[5].ctypes.data_as(C.POINTER(C.c_int))
            tr.final_x = C.POINTER(C.c_double)()
            self._raw = (key, bufs, tr)
        tr = self._raw[2]
        co = opts.to_c()
        rc = _capi.lib().coopcg_gpu_run(self._h, C.byref(co), C.byref(tr))
        _check(self._h, rc)
        _capi.lib().coopcg_gpu_timing(self._h, C.byref(self._timing))
        return tr.iterations, tr.exact_rank_checks

    def _make_trace(self, tr, norms, minres, wall, init, fres, fx, opts, act=None) -> SolveTrace:
        n, p = self.n, self.p
        it = tr.iterations
        every = opts.recompute_residual_every if opts.recompute_residual_every >= 0 else 50
        recs = []
        for k in range(it):
            rc = every > 0 and (k + 1) % every == 0
            agents = [j for j in range(p) if not np.isnan(norms[k, j])]
            pk = len(agents)
            m = iteration_mults(n, pk, rc)
            recs.append(IterationRecord(k=k, active_agents=pk, agents=agents,
                                        residual_norms=norms[k, agents].copy(), minres=float(minres[k]),
                                        mults=m, mults_per_worker=[m] * pk, wall_ns=int(wall[k])))
        active = [int(a) for a in act[:tr.n_active]] if act is not None else list(range(p))
        return SolveTrace(iterations=recs, status=TerminalStatus(tr.status),
                          converged_agent=tr.converged_agent,
                          final_x=(fx.T[:, active].copy() if fx is not None else None),
                          active_agents=active, initial_residual_norms=init,
                          initial_minres=tr.initial_minres, final_residual_norms=fres[active].copy(),
                          final_minres=tr.final_minres, setup_mults=n * n,
                          final_residual_norms_by_id=fres.copy(),
                          loop_wall_ns=int(tr.loop_wall_ns), residual_norms=norms[:it].copy(),
                          minres=minres[:it].copy(), wall_ns=wall[:it].copy(),
                          exact_rank_checks=tr.exact_rank_checks)

    def solve(self, b, X0, opts: Optional[SolveOptions] = None) -> SolveTrace:
        self.upload(b, X0)
        return self.run(opts)

    def timing(self) -> dict:
        """coopcg_timing of the last solve (run / run_raw / the phase API's end)."""
        _capi.lib().coopcg_gpu_timing(self._h, C.byref(self._timing))
        t = self._timing
        return {"matvec_launches": t.matvec_launches, "matvec_ms_total": t.matvec_ms_total,
                "run_ms": t.run_ms, "loop_ms": t.loop_ms, "kernel_launches": t.kernel_launches,
                "a_l2_resident_bytes": t.a_l2_resident_bytes}

    def stream_handle(self) -> int:
        """cudaStream_t of this context (for events on the launching stream)."""
        return int(_capi.lib().coopcg_gpu_stream(self._h) or 0)

    # -- kernel-level entry points --
    def matvec_block(self, D: np.ndarray) -> np.ndarray:
        D = np.asarray(D, dtype=np.float64)
        if D.shape != (self.n, self.p):
            raise DimensionError("matvec_block: row count does not match matrix dimension")
        Dc = np.ascontiguousarray(D.T)
        out = np.zeros((self.p, self.row_end - self.row_begin))
        _check(self._h, _capi.lib().coopcg_gpu_matvec_block(self._h, Dc.ctypes.data, out.ctypes.data))
        return out.T.copy()

    def numerical_rank(self, D: np.ndarray, tol: float, force_exact: bool = False) -> int:
        D = np.asarray(D, dtype=np.float64)
        if D.shape != (self.n, self.p):
            raise DimensionError("numerical_rank: shape")
        Dc = np.ascontiguousarray(D.T)
        r = C.c_int()
        _check(self._h, _capi.lib().coopcg_gpu_numerical_rank_ex(self._h, Dc.ctypes.data, tol,
                                                                 1 if force_exact else 0, C.byref(r)))
        return r.value


def ccg_solve(A: np.ndarray, b: np.ndarray, X0: np.ndarray, opts: Optional[SolveOptions] = None,
              gpu: Optional[GpuOptions] = None) -> SolveTrace:
    """Cooperative block CG on the GPU with ccg_solve's semantics
    (coopcg/solvers.hpp:325-333).  A is (n, n), b (n,), X0 (n, p)."""
    gpu = gpu or GpuOptions()
    A = np.asarray(A, dtype=np.float64)
    X0 = np.asarray(X0, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise DimensionError("SpdMatrix: entry grid does not match dimension")
    n = A.shape[0]
    if b.shape != (n,) or X0.ndim != 2 or X0.shape[0] != n:
        raise DimensionError("solver: operand shapes do not match the system matrix")
    p = X0.shape[1]
    if p < 1 or p >= n:
        raise DimensionError("solver: need 1 <= p < n starting columns")
    with GpuContext(n, p, gpu.device, gpu.arith, devices=gpu.devices) as ctx:
        ctx.set_A(A)
        return ctx.solve(b, X0, opts)


def _single_vector_solve(A, b, x0, opts, gpu, algo):
    import dataclasses
    gpu = gpu or GpuOptions()
    opts = opts or SolveOptions()
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    x0 = np.asarray(x0, dtype=np.float64)
    n = A.shape[0]
    if A.shape != (n, n) or b.shape != (n,) or x0.shape != (n,):
        raise DimensionError(f"{'cg_solve' if algo == 'ccg' else 'steepest_descent_solve'}: "
                             "operand shapes do not match")
    every = opts.recompute_residual_every if opts.recompute_residual_every >= 0 else 1
    o = dataclasses.replace(opts, recompute_residual_every=every, algo=algo)
    name = "cg_solve" if algo == "ccg" else "steepest_descent_solve"
    with GpuContext(n, 1, gpu.device, gpu.arith if algo == "ccg" else "exact") as ctx:
        ctx.set_A(A)
        try:
            t = ctx.solve(b, x0[:, None], o)
        except SpdViolationError as ex:  # the scalar solvers' own text (solvers.hpp:448-449, :583-585)
            k = str(ex).rsplit(" ", 1)[-1]
            what = "direction" if algo == "ccg" else "gradient"
            raise SpdViolationError(f"{name}: nonpositive {what} energy at iteration {k}") from None
    # the scalar solvers' own counting (solvers.hpp:438-486, :571-603)
    for rec in t.iterations:
        rc = every > 0 and (rec.k + 1) % every == 0
        if algo == "ccg":
            m = (2 * n * n + 5 * n + 2) if rc else (n * n + 6 * n + 2)
        else:
            m = (2 * n * n + 3 * n + 1) if rc else (n * n + 4 * n + 1)
        rec.mults = m
        rec.mults_per_worker = [m]
    return t


def cg_solve(A, b, x0, opts: Optional[SolveOptions] = None, gpu: Optional[GpuOptions] = None) -> SolveTrace:
    """Classical CG (solvers.hpp:388-530) on the block kernels: the p = 1 block
    solver with the same residual policy (default: recompute every step)
    reproduces cg_solve bit for bit (tests/test_solvers.cpp:176-201)."""
    return _single_vector_solve(A, b, x0, opts, gpu, "ccg")


def steepest_descent_solve(A, b, x0, opts: Optional[SolveOptions] = None,
                           gpu: Optional[GpuOptions] = None) -> SolveTrace:
    """Steepest descent (solvers.hpp:532-646): p = 1 with beta = 0 (exact mode)."""
    return _single_vector_solve(A, b, x0, opts, gpu, "sd")


# ---- host generators for b, X0 -------------------------------
def gen_rhs(n: int, kind: str, seed: int) -> np.ndarray:
    b = np.zeros(n)
    _check(None, _capi.lib().coopcg_gen_rhs(n, 0 if kind == "uniform" else 1, seed, b.ctypes.data))
    return b


def gen_starts(n: int, p: int, seed: int) -> np.ndarray:
    X0c = np.zeros((p, n))
    _check(None, _capi.lib().coopcg_gen_starts(n, p, seed, X0c.ctypes.data))
    return X0c.T.copy()


def gen_random_spd_spectrum(n: int, cond: float, seed: int) -> np.ndarray:
    """The spectrum of random_spd_with_spectrum (problem.hpp:125-139)."""
    lam = np.zeros(n)
    _check(None, _capi.lib().coopcg_gen_random_spd_spectrum(n, cond, seed, lam.ctypes.data))
    return lam


def gen_reference_rhs_starts(n: int, p: int, seed: int):
    """random_rhs_and_starts<double> (problem.hpp:187-200): b, X0 ~ U[-10, 10]."""
    b = np.zeros(n)
    X0c = np.zeros((p, n))
    _check(None, _capi.lib().coopcg_gen_reference_rhs_starts(n, p, seed, b.ctypes.data, X0c.ctypes.data))
    return b, X0c.T.copy()


def gen_householder_factors(n: int, m: int, kappa: float, seed: int):
    V = np.zeros((max(m, 1), n))
    lam = np.zeros(n)
    _check(None, _capi.lib().coopcg_gen_householder_factors(n, m, kappa, seed, V.ctypes.data,
                                                              lam.ctypes.data))
    return V[:m], lam


def row_split(n: int, parts: int, part: int) -> tuple:
    """The library's row blocks (coopcg_row_split): rows [r0, r1) of shard `part`."""
    r0, r1 = C.c_int(), C.c_int()
    _check(None, _capi.lib().coopcg_row_split(n, parts, part, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for GpuContext(..., nccl=(nranks, rank, id))."""
    buf = C.create_string_buffer(_capi.NCCL_ID_BYTES)
    _check(None, _capi.lib().coopcg_nccl_unique_id(buf))
    return buf.raw


def library_version() -> str:
    return _capi.lib().coopcg_gpu_version().decode()
