"""Parity at the full BASELINE configs (BASELINE.json configs 1-4, SURVEY.md
§8d), against the reference itself on identical bytes.

The reference is oracle/_ref/libccgref.so: the unmodified reference headers
compiled by oracle/Makefile, run as parallel_ccg (coopcg/parallel.hpp:76-111,
one OpenMP thread per agent -- bitwise equal to ccg_solve, solvers.hpp:329-333,
tests/test_oracle.py).  For each config:

  1. A is generated on the HOST by the oracle's generator (oracle/gen_oracle.c,
     OpenMP over rows, same bits as the serial restatement) straight into a
     matrix the reference shim owns (one host copy: 2.1 / 34 / 137 GB at
     cfg 2 / 3 / 4; the box host has 196 GB);
  2. the product generates A on the DEVICE (coopcg_gpu_gen_A) and every row is
     compared with the host copy, bit for bit (this pins the device generators
     at full size, the Householder one at n = 65536 included);
  3. the product solves in exact mode and in fast mode on its device A with
     b / X0 from the oracle's generators;
  4. the reference solves on the host copy.

Exact mode must be bit-identical: status, iteration count, converged agent,
initial norms, every per-iteration per-agent recurrence norm, minres, final X,
the true final residual norms.  Fast mode (north star): X within 1e-8
relative; the residual-norm history within 1e-8 relative for k < k_div
(tests/golden/kdiv.json: where the reference's own FMA-contracted build
leaves the 1e-8 band or the history reaches the round-off floor); iteration
count to tolerance within +-2 (cfg 1).

Iterations: cfg 1 the full solve to 1e-10 ||b|| (~1.1k iterations), cfg 2 all
200 fixed iterations, cfg 3 / cfg 4 setup + 4 / 2 iterations + finalize (the
reference streams A once per agent per iteration: 4.3 s per iteration at
cfg 3 and 41 s at cfg 4 with its one-thread-per-agent OpenMP team on the box's
16 cores).  Its finalize_trace recomputes the p true residuals one agent after
another in the coordinator (solvers.hpp:188-210): ~9 minutes of latency-bound
matvecs at cfg 4.  At cfg 3 / 4 the test therefore runs parallel_ccg with that
per-agent loop executed by the team, agent j on worker j, with the reference's
own matvec_col / norm2 (oracle/ref_shim.cpp, parallel_ccg_team_finalize; every
other step is the reference's drive() and OmpExecutor) -- bit-identical to
parallel_ccg (tests/test_oracle.py::test_team_finalize_equals_parallel_ccg).
A summary (times, deltas) is written to gpurun_out/full_config_parity.json.
"""
import json
import os
import time

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ITERS = {1: None, 2: None, 3: 4, 4: 2}   # None: the config's own stopping rule
KDIV = json.load(open(os.path.join(ROOT, "tests", "golden", "kdiv.json")))
SUMMARY = os.path.join(ROOT, "gpurun_out", "full_config_parity.json")


@pytest.fixture(scope="module")
def m():
    import paper_1204_0069_b200 as mod
    with mod.GpuContext(8, 2) as _:
        pass
    return mod


def _host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_AVPHYS_PAGES")
    except (ValueError, OSError):
        return 0


def _record(key, value):
    os.makedirs(os.path.dirname(SUMMARY), exist_ok=True)
    d = json.load(open(SUMMARY)) if os.path.exists(SUMMARY) else {}
    d[key] = value
    json.dump(d, open(SUMMARY, "w"), indent=1, sort_keys=True)


def _compare_A(ctx, R, n, rows_per_slice):
    buf = np.empty((rows_per_slice, n))
    for r0 in range(0, n, rows_per_slice):
        k = min(rows_per_slice, n - r0)
        got = ctx.get_A(r0, k, out=buf[:k])
        if not np.array_equal(got, R.A[r0:r0 + k]):
            bad = np.argwhere(got != R.A[r0:r0 + k])[0]
            raise AssertionError(f"device A differs from the oracle generator at row {r0 + bad[0]}, col {bad[1]}")


def _rel_x(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.maximum(np.linalg.norm(b, axis=0), 1e-300)))


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_full_config_parity(m, po, c):
    cfg = m.CONFIGS[c]
    n, p = cfg.n, cfg.p
    need = 8.0 * n * n + 8e9
    if _host_ram_bytes() and _host_ram_bytes() < need:
        pytest.skip(f"host RAM {_host_ram_bytes() / 1e9:.0f} GB < {need / 1e9:.0f} GB for the reference's copy of A")
    times = {}
    t0 = time.time()
    R = po.RefMatrix(n)
    try:
        if cfg.matrix == "diagdom":
            po.gen_diagdom_rows(n, cfg.seed, 0, n, out=R.A)
        else:
            po.gen_householder_into(n, cfg.reflectors, cfg.kappa, cfg.seed, R.A)
        times["host_gen_s"] = time.time() - t0
        b = po.gen_rhs(n, cfg.rhs, cfg.seed)
        X0 = po.gen_starts(n, p, cfg.seed)
        nb = po.seq_norm(b)
        tol = cfg.rel_tol * nb if cfg.fixed_iters < 0 else 0.0
        max_iters = ITERS[c] if ITERS[c] is not None else cfg.fixed_iters
        opts = m.SolveOptions(tol=tol, max_iters=max_iters)
        rows_per_slice = max(1, (256 << 20) // (8 * n))

        gt = {}
        for arith in ("exact", "fast"):
            t0 = time.time()
            with m.GpuContext(n, p, arith=arith) as ctx:
                ctx.gen_A(cfg.matrix, cfg.seed, cfg.reflectors, cfg.kappa)
                if arith == "exact":
                    _compare_A(ctx, R, n, rows_per_slice)
                else:  # the fast layout's round trip: first and last slices
                    for r0 in (0, max(0, n - rows_per_slice)):
                        k = min(rows_per_slice, n - r0)
                        assert np.array_equal(ctx.get_A(r0, k), R.A[r0:r0 + k])
                times[f"{arith}_gen_and_compare_s"] = time.time() - t0
                t0 = time.time()
                gt[arith] = ctx.solve(b, X0, opts)
                times[f"{arith}_solve_s"] = time.time() - t0

        t0 = time.time()
        # cfg 3 / 4: parallel_ccg with finalize_trace's agent loop on the team
        # (bit-identical, tests/test_oracle.py::test_team_finalize_equals_parallel_ccg)
        algo = "parallel_team_finalize" if c >= 3 else "parallel"
        ot = R.solve(b, X0, tol=tol, max_iters=max_iters, algo=algo)
        times["reference_solve_s"] = time.time() - t0
    finally:
        R.close()
    assert ot.rc == 0, ot.error

    # exact: bit for bit
    e = gt["exact"]
    assert str(e.status) == ot.status
    assert e.iteration_count() == ot.iterations
    assert e.converged_agent == ot.converged_agent
    assert np.array_equal(e.initial_residual_norms, ot.initial_residual_norms)
    assert np.array_equal(e.residual_norms, ot.residual_norms)
    assert np.array_equal(e.minres, ot.minres)
    assert np.array_equal(e.final_x, ot.final_x)
    assert np.array_equal(e.final_residual_norms, ot.final_residual_norms)
    assert e.final_minres == ot.final_minres

    # fast: the north star's tolerances
    f = gt["fast"]
    kd = KDIV.get(f"cfg{c}", {}).get("k_div", ot.iterations)
    k = min(f.iteration_count(), ot.iterations, kd)
    hist = np.abs(f.residual_norms[:k] - ot.residual_norms[:k]) / ot.residual_norms[:k]
    hist_max = float(hist.max()) if k else 0.0
    xrel = _rel_x(f.final_x, ot.final_x)
    d_it = f.iteration_count() - ot.iterations
    wall = ot.wall_ns.astype(np.float64)
    # true final residuals: within 1e-8 relative where above the round-off floor
    above = ot.final_residual_norms / nb > 1e-11
    fres = np.abs(f.final_residual_norms - ot.final_residual_norms) / ot.final_residual_norms
    fres_max = float(fres[above].max()) if above.any() else 0.0
    _record(f"cfg{c}", {
        "n": n, "p": p, "iterations": ot.iterations, "status": ot.status,
        "exact": "bit-identical", "fast_delta_iterations": d_it, "fast_x_rel": xrel,
        "fast_history_max_rel_k_lt_kdiv": hist_max, "k_div": kd, "fast_status": str(f.status),
        "fast_final_residual_rel": float(np.max(f.final_residual_norms / nb)),
        "fast_final_residual_vs_reference_rel_above_floor": fres_max,
        "reference_s_per_iteration": float(np.mean(wall) * 1e-9) if len(wall) else None,
        "reference_threads": p, "host_cores": os.cpu_count(), "reference_entry": algo, "times_s": times})
    assert str(f.status) == ot.status
    assert abs(d_it) <= 2
    assert hist_max < 1e-8
    assert xrel < 1e-8
    if kd >= ot.iterations:
        # the whole history is inside the comparable band (cfg 3 / 4): the true
        # final residuals agree like the history does
        assert fres_max < 1e-8
    else:
        # past k_div (cfg 1 converged to tol, cfg 2 at the round-off floor) the
        # two runs' last iterates differ at the rounding level of their own
        # residual: both true residuals are that small
        assert np.all(f.final_residual_norms <= 10 * np.maximum(ot.final_residual_norms, 1e-11 * nb))
