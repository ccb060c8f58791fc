#!/usr/bin/env python3
"""Randomised parity sweep on the GPU box (test infrastructure, not product).

Draws solver cases -- n (biased to the panel / tile / wave boundaries of the
kernels), p in 1..32, matrix family, stopping rule, residual-recompute policy,
algorithm (ccg / mccg), one context or 2-3 row shards -- and compares the
device solve with the compiled reference (oracle/_ref/libccgref.so):

  exact mode: bit for bit (status, iteration count, converged agent, every
              per-iteration per-agent norm, final X, true final residuals,
              and the error class when the reference throws);
  fast mode:  final X within 1e-8 relative when both converge, iteration
              count within +-2 on the diagonally dominant family, same status.

    python tools/fuzz_parity.py --seconds 300 --seed 1 [--out gpurun_out/fuzz.json]

Every case is reproducible from the printed (seed, index).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
os.environ.setdefault("OMP_WAIT_POLICY", "passive")

RANK_SHARE = 0.0  # --rank-share: fraction of the exact sessions run on a rank context (NCCL path)
EDGES = [31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 287, 288, 289, 511, 512, 513, 1023, 1024, 1025]


def draw_case(rng, multi=False, large=False):
    p = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 9, 12, 15, 16, 17, 24, 31, 32]))
    kind = rng.choice(["edge", "small", "mid"], p=[0.4, 0.3, 0.3])
    if large:  # --large: the A.D variants picked above 148 * 64 local rows, a few iterations each
        p = int(rng.choice([3, 4, 7, 8, 13, 16, 24, 32]))
        n = int(rng.choice([9471, 9472, 9473, 9600, 10240, 11000, 12289])) + int(rng.integers(-1, 2))
        return dict(n=n, p=p, matrix=str(rng.choice(["diagdom", "householder"])), kappa=float(10 ** rng.uniform(1, 4)),
                    m=int(rng.integers(1, 5)), max_iters=int(rng.integers(1, 4)), tol_rel=0.0,
                    recompute=int(rng.choice([-1, 1, 2])), algo="ccg", shards=int(rng.choice([1, 1, 2])),
                    degenerate=False, seed=int(rng.integers(1, 2**31)))
    if kind == "edge":
        n = int(rng.choice(EDGES)) + int(rng.integers(-1, 2))
    elif kind == "small":
        n = int(rng.integers(p + 1, 200))
    else:
        n = int(rng.integers(200, 2600))
    n = max(n, p + 1, 2)
    matrix = str(rng.choice(["diagdom", "householder", "random_spd"], p=[0.5, 0.3, 0.2]))
    if matrix == "random_spd" and n > 700:
        matrix = "diagdom"  # the reference's O(n^3) generator
    kappa = float(10 ** rng.uniform(0.5, 4.5))
    m = int(rng.integers(1, 9))
    fixed = bool(rng.random() < 0.4)
    max_iters = int(rng.integers(0, 45)) if fixed else -1
    tol_rel = 0.0 if fixed else float(10 ** rng.uniform(-12, -6))
    recompute = int(rng.choice([-1, 0, 1, 2, 3, 7, 50]))
    algo = str(rng.choice(["ccg", "mccg"], p=[0.8, 0.2]))
    shards = int(rng.choice([1, 1, 2, 3])) if n >= 200 else 1
    if multi:  # --multi: row shards only, long ill-conditioned runs
        n = max(n, 200)
        shards = int(rng.choice([2, 3, 4]))
        matrix = "householder" if rng.random() < 0.8 else "diagdom"
        algo = "mccg" if rng.random() < 0.25 else "ccg"
    degenerate = bool(rng.random() < 0.06) and p > 1
    return dict(n=n, p=p, matrix=matrix, kappa=kappa, m=m, max_iters=max_iters, tol_rel=tol_rel,
                recompute=recompute, algo=algo, shards=shards, degenerate=degenerate,
                seed=int(rng.integers(1, 2**31)))


def cost(c):
    its = c["max_iters"] if c["max_iters"] >= 0 else 2 * c["n"]  # worst case: the run reaches max_iters = 2n
    return float(c["n"]) ** 2 * c["p"] * max(its, 1)


def run_case(m, po, c, arith):
    n, p = c["n"], c["p"]
    if c["matrix"] == "diagdom":
        A = po.gen_diagdom(n, c["seed"])
        b = po.gen_rhs(n, "uniform", c["seed"])
    elif c["matrix"] == "householder":
        A = po.gen_householder(n, c["m"], c["kappa"], c["seed"])
        b = po.gen_rhs(n, "normal", c["seed"])
    else:
        A, b, _ = po.ref_make_problem(n, p, c["kappa"], c["seed"])
    X0 = po.gen_starts(n, p, c["seed"])
    if c["degenerate"]:
        X0[:, -1] = X0[:, 0]  # duplicate start: rank-deficient D0 (ccg: collapse at k = 0; mccg restricts)
    tol = c["tol_rel"] * po.seq_norm(b)
    ref = po.ref_solve(A, b, X0, tol=tol, max_iters=c["max_iters"], recompute=c["recompute"], algo=c["algo"])
    opts = m.SolveOptions(tol=tol, max_iters=c["max_iters"], recompute_residual_every=c["recompute"],
                          algo=c["algo"])
    gpu = m.GpuOptions(arith=arith, devices=[0] * c["shards"] if c["shards"] > 1 else None)
    try:
        t = m.ccg_solve(A, b, X0, opts, gpu)
        err = None
    except m.Error as ex:
        t, err = None, ex
    if ref.rc != 0 or err is not None:
        # the reference threw: same class of failure (pyoracle rc: 2 SPD violation, 3 breakdown)
        want = {2: m.SpdViolationError, 3: m.NumericalBreakdownError}.get(ref.rc)
        if arith == "exact":
            if want is None or not isinstance(err, want):
                return f"error mismatch: reference rc={ref.rc} ({ref.error!r}), device {err!r}"
        return None
    if arith == "exact":
        if str(t.status) != ref.status or t.iteration_count() != ref.iterations:
            return f"status/iterations {t.status}/{t.iteration_count()} vs {ref.status}/{ref.iterations}"
        if t.converged_agent != ref.converged_agent:
            return "converged agent"
        if not np.array_equal(t.residual_norms, ref.residual_norms, equal_nan=True):
            return "per-iteration norms differ"
        if list(t.active_agents) != list(ref.extra["active_agents"]):
            return "active agents differ"
        act = list(t.active_agents)
        if not np.array_equal(t.final_x, ref.final_x[:, act], equal_nan=True):
            return "final X differs"
        if not np.array_equal(t.final_residual_norms, ref.final_residual_norms[act], equal_nan=True):
            return "final residual norms differ"
        return None
    # fast mode (the north star's tolerances); mccg restrictions and rank-collapse exits depend
    # on rounding-level rank decisions, so only converged ccg runs are held to them -- and only
    # while the block Krylov space is not exhausted (iterations * p well below n: past that the
    # direction block loses rank in exact arithmetic and the exit is decided by rounding)
    if c["algo"] != "ccg" or ref.status != "converged" or ref.iterations * c["p"] > 0.8 * c["n"]:
        return None
    if str(t.status) != "converged":
        return f"fast status {t.status} vs converged"
    rel = float(np.max(np.linalg.norm(t.final_x - ref.final_x, axis=0) /
                       np.maximum(np.linalg.norm(ref.final_x, axis=0), 1e-300)))
    cond = c["kappa"] if c["matrix"] != "diagdom" else 2.0
    if rel > max(1e-8, 10 * cond * c["tol_rel"]):
        return f"fast X rel diff {rel:.2e} (cond {cond:.1e}, tol_rel {c['tol_rel']:.1e})"
    if c["matrix"] == "diagdom" and abs(t.iteration_count() - ref.iterations) > 2:
        return f"fast iterations {t.iteration_count()} vs {ref.iterations}"
    return None


def run_misc(m, po, rng):
    """The other entry points on random shapes, bit for bit: the scalar solvers against the
    reference's cg_solve / steepest_descent_solve, the device generators against the oracle's,
    matvec_block and numerical_rank (certificate and forced-exact paths) against the reference."""
    what = str(rng.choice(["cg", "sd", "gen", "matvec", "rank"]))
    seed = int(rng.integers(1, 2**31))
    if what in ("cg", "sd"):
        n = int(rng.integers(3, 400))
        A = po.gen_diagdom(n, seed) if rng.random() < 0.4 else po.gen_householder(
            n, int(rng.integers(1, 6)), float(10 ** rng.uniform(0.3, 3.5)), seed)
        b = po.gen_rhs(n, "normal", seed)
        x0 = po.gen_starts(n, 1, seed)[:, 0] if rng.random() < 0.7 else np.zeros(n)
        fixed = rng.random() < 0.4
        mi = int(rng.integers(0, 50)) if fixed else -1
        tol = 0.0 if fixed else float(10 ** rng.uniform(-11, -5)) * po.seq_norm(b)
        rec = int(rng.choice([-1, 0, 1, 2, 5]))
        ref = po.ref_cg(A, b, x0, tol=tol, max_iters=mi, recompute=rec, algo=what)
        fn = m.cg_solve if what == "cg" else m.steepest_descent_solve
        try:
            t = fn(A, b, x0, m.SolveOptions(tol=tol, max_iters=mi, recompute_residual_every=rec))
        except m.Error as ex:
            return None if ref.rc != 0 else f"{what} n={n} seed={seed}: device raised {ex!r}"
        if ref.rc != 0:
            return f"{what} n={n} seed={seed}: reference raised {ref.error!r}, device did not"
        ok = (str(t.status) == ref.status and t.iteration_count() == ref.iterations and
              np.array_equal(t.residual_norms, ref.residual_norms) and np.array_equal(t.final_x, ref.final_x) and
              np.array_equal(t.final_residual_norms, ref.final_residual_norms))
        return None if ok else f"{what} n={n} seed={seed} mi={mi} rec={rec}: differs from the reference"
    p = int(rng.choice([1, 2, 3, 4, 7, 8, 9, 16, 17, 31, 32]))
    n = max(p + 1, int(rng.choice(EDGES)) + int(rng.integers(-1, 2)) if rng.random() < 0.5 else int(rng.integers(p + 1, 3000)))
    arith = str(rng.choice(["exact", "fast"]))
    shards = int(rng.choice([1, 1, 2, 3])) if n >= 200 else 1
    with m.GpuContext(n, p, arith=arith, devices=[0] * shards if shards > 1 else None) as ctx:
        if what == "gen":
            if rng.random() < 0.5:
                ctx.gen_A("diagdom", seed)
                want = po.gen_diagdom(n, seed)
            else:
                mr, kap = int(rng.integers(1, 9)), float(10 ** rng.uniform(0.3, 6))
                ctx.gen_A("householder", seed, mr, kap)
                want = po.gen_householder(n, mr, kap, seed)
            return None if np.array_equal(ctx.get_A(), want) else f"gen n={n} p={p} {arith} shards={shards} seed={seed}"
        if what == "matvec":
            A = po.gen_diagdom(n, seed)
            ctx.set_A(A)
            D = np.random.default_rng(seed).uniform(-1, 1, (n, p))
            Q = ctx.matvec_block(D)
            ref = np.zeros((p, n))
            Dc = np.ascontiguousarray(D.T)
            po.oracle_lib().orc_matvec_block(A.ctypes.data, n, Dc.ctypes.data, p, ref.ctypes.data)
            if arith == "exact":
                return None if np.array_equal(Q, ref.T) else f"matvec n={n} p={p} shards={shards} seed={seed}"
            err = np.max(np.abs(Q - ref.T) / (np.abs(A) @ np.abs(D)))
            return None if err < 1e-14 else f"fast matvec n={n} p={p} shards={shards} seed={seed}: {err:.1e}"
        # numerical_rank: full rank, a duplicated / scaled column, a zero column, badly scaled columns
        if shards > 1:
            return None
        g = np.random.default_rng(seed)
        D = g.standard_normal((n, p)) * 10.0 ** g.integers(-6, 7, size=p)
        kind = int(g.integers(0, 4))
        if p > 1 and kind == 1:
            D[:, -1] = 2.0 * D[:, 0]
        elif kind == 2:
            D[:, int(g.integers(0, p))] = 0.0
        elif p > 2 and kind == 3:
            D[:, 1] = D[:, 0] + 1e-9 * D[:, 2]
        want, _ = po.numerical_rank(D, 1e-10, lib="ref")
        for force in (False, True):
            got = ctx.numerical_rank(D, 1e-10, force_exact=force)
            if got != want:
                return f"rank n={n} p={p} {arith} kind={kind} force={force} seed={seed}: {got} vs {want}"
    return None


def run_session_fast(m, po, rng):
    """Fast mode: 3-5 solves on one resident context (ccg / mccg, changing options) must
    each equal, bit for bit, the same solve on a fresh context -- nothing may carry over."""
    p = int(rng.choice([1, 2, 3, 4, 6, 8, 9, 16, 17, 32]))
    n = int(rng.integers(max(p + 2, 20), 700))
    seed = int(rng.integers(1, 2**31))
    A = po.gen_diagdom(n, seed) if rng.random() < 0.5 else po.gen_householder(
        n, int(rng.integers(1, 6)), float(10 ** rng.uniform(0.5, 3.0)), seed)
    shards = int(rng.choice([1, 1, 2, 3])) if n >= 200 else 1
    gpu = m.GpuOptions(arith="fast", devices=[0] * shards if shards > 1 else None)
    log = []
    with m.GpuContext(n, p, arith="fast", devices=gpu.devices) as ctx:
        ctx.set_A(A)
        for step in range(int(rng.integers(3, 6))):
            s2 = int(rng.integers(1, 2**31))
            b = po.gen_rhs(n, "uniform", s2)
            X0 = po.gen_starts(n, p, s2)
            if p > 1 and rng.random() < 0.25:
                X0[:, -1] = X0[:, 0]
            fixed = rng.random() < 0.5
            opts = m.SolveOptions(tol=0.0 if fixed else float(10 ** rng.uniform(-10, -6)) * po.seq_norm(b),
                                  max_iters=int(rng.integers(0, 70)) if fixed else -1,
                                  recompute_residual_every=int(rng.choice([-1, 0, 1, 3, 7])),
                                  algo="mccg" if (rng.random() < 0.3 and shards == 1) else "ccg")
            log.append(dict(step=step, n=n, p=p, shards=shards, seed=s2, max_iters=opts.max_iters, tol=opts.tol,
                            rec=opts.recompute_residual_every, algo=opts.algo))
            res = []
            for fresh in (False, True):
                try:
                    t = m.ccg_solve(A, b, X0, opts, gpu) if fresh else ctx.solve(b, X0, opts)
                    res.append((str(t.status), t.iteration_count(), t.residual_norms.tobytes(), t.final_x.tobytes()))
                except m.Error as ex:
                    res.append((type(ex).__name__, str(ex)))
            if res[0] != res[1]:
                return f"{log}: resident {res[0][:2]} vs fresh {res[1][:2]}"
    return None


def run_session(m, po, rng):
    """3-6 solves on one resident context: new b / X0, ccg / mccg, growing and shrinking
    max_iters, every recompute policy, verification mode on and off, both arithmetic
    modes' contexts -- each exact solve bit for bit against the reference."""
    p = int(rng.choice([1, 2, 3, 4, 6, 8, 9, 16, 17, 32]))
    n = int(rng.integers(max(p + 2, 20), 500))
    seed = int(rng.integers(1, 2**31))
    if rng.random() < 0.5:
        A = po.gen_diagdom(n, seed)
    else:
        A = po.gen_householder(n, int(rng.integers(1, 6)), float(10 ** rng.uniform(0.5, 3.5)), seed)
    shards = int(rng.choice([1, 1, 1, 2])) if n >= 200 else 1
    rank_ctx = shards == 1 and rng.random() < RANK_SHARE  # a rank context (NCCL exchanges, world of one)
    log = []
    kw = dict(nccl=(1, 0, m.nccl_unique_id())) if rank_ctx else dict(devices=[0] * shards if shards > 1 else None)
    with m.GpuContext(n, p, **kw) as ctx:
        ctx.set_A(A)
        for step in range(int(rng.integers(3, 7))):
            s2 = int(rng.integers(1, 2**31))
            b = po.gen_rhs(n, "uniform" if rng.random() < 0.5 else "normal", s2)
            X0 = po.gen_starts(n, p, s2)
            if p > 1 and rng.random() < 0.25:
                X0[:, -1] = X0[:, 0]
            fixed = rng.random() < 0.5
            max_iters = int(rng.integers(0, 60)) if fixed else -1
            tol = 0.0 if fixed else float(10 ** rng.uniform(-11, -6)) * po.seq_norm(b)
            rec = int(rng.choice([-1, 0, 1, 3, 7]))
            algo = "mccg" if rng.random() < 0.3 else "ccg"
            verify = (shards == 1 and not rank_ctx and algo == "ccg" and rng.random() < 0.3 and
                      (max_iters >= 0 or n <= 200))
            xs = np.linalg.solve(A, b) if verify else None
            log.append(dict(step=step, n=n, p=p, shards=shards, rank_ctx=bool(rank_ctx), seed=s2, max_iters=max_iters,
                            tol=tol, rec=rec, algo=algo, verify=bool(verify)))
            ref = po.ref_solve(A, b, X0, tol=tol, max_iters=max_iters, recompute=rec, algo=algo)
            opts = m.SolveOptions(tol=tol, max_iters=max_iters, recompute_residual_every=rec, algo=algo,
                                  keep_history=bool(verify), x_star=xs)
            try:
                t = ctx.solve(b, X0, opts)
                err = None
            except m.Error as ex:
                t, err = None, ex
            if ref.rc != 0 or err is not None:
                want = {2: m.SpdViolationError, 3: m.NumericalBreakdownError}.get(ref.rc)
                if want is None or not isinstance(err, want):
                    return f"{log}: error mismatch: reference rc={ref.rc} ({ref.error!r}), device {err!r}"
                continue
            act = list(t.active_agents)
            ok = (str(t.status) == ref.status and t.iteration_count() == ref.iterations and
                  np.array_equal(t.residual_norms, ref.residual_norms, equal_nan=True) and
                  act == list(ref.extra["active_agents"]) and
                  np.array_equal(t.final_x, ref.final_x[:, act], equal_nan=True) and
                  np.array_equal(t.final_residual_norms, ref.final_residual_norms[act], equal_nan=True))
            if not ok:
                return f"{log}: solve differs from the reference ({t.status}/{t.iteration_count()} vs {ref.status}/{ref.iterations})"
            if verify:
                if len(t.history_x) != t.iteration_count() + 1 or not np.array_equal(t.history_x[-1], t.final_x):
                    return f"{log}: history entries"
                if t.iteration_count() and t.iterations[-1].anorm_errors is None:
                    return f"{log}: anorm missing"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-cost", type=float, default=3e9)
    ap.add_argument("--multi", action="store_true", help="row-sharded cases only (2-4 shards), mostly Householder")
    ap.add_argument("--large", action="store_true", help="n around 9472..12290 (the large-n A.D variants), 1-3 iterations")
    ap.add_argument("--rank-share", type=float, default=0.0,
                    help="--session: share of the sessions on a coopcg_gpu_create_rank context (world of one)")
    ap.add_argument("--misc", action="store_true",
                    help="scalar solvers, device generators, matvec_block, numerical_rank on random shapes")
    ap.add_argument("--session", nargs="?", const="exact", default="", choices=["exact", "fast"],
                    help="several solves with changing options on ONE resident context (state carried between "
                         "solves): exact against the reference, fast against the same solve on a fresh context")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_1204_0069_b200 as m
    import pyoracle as po
    global RANK_SHARE
    RANK_SHARE = args.rank_share
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    done = {"exact": 0, "fast": 0}
    failures = []
    idx = 0
    while time.time() - t0 < args.seconds:
        if args.misc:
            idx += 1
            try:
                why = run_misc(m, po, rng)
            except Exception as ex:
                why = f"exception {type(ex).__name__}: {ex}"
            done["exact"] += 1
            if why:
                failures.append({"index": idx, "arith": "misc", "why": why})
                print(f"FAIL misc #{idx}: {why}", flush=True)
            continue
        if args.session:
            idx += 1
            why = run_session_fast(m, po, rng) if args.session == "fast" else run_session(m, po, rng)
            done["exact"] += 1
            if why:
                failures.append({"index": idx, "arith": "session", "why": why})
                print(f"FAIL session #{idx}: {why}", flush=True)
            continue
        c = draw_case(rng, args.multi, args.large)
        idx += 1
        if cost(c) > args.max_cost:
            continue
        for arith in ("exact", "fast"):
            try:
                why = run_case(m, po, c, arith)
            except Exception as ex:  # a crash is a failure of the case, not of the sweep
                why = f"exception {type(ex).__name__}: {ex}"
            done[arith] += 1
            if why:
                failures.append({"index": idx, "arith": arith, "case": c, "why": why})
                print(f"FAIL #{idx} {arith} {c}: {why}", flush=True)
    res = {"seed": args.seed, "seconds": round(time.time() - t0, 1), "cases_drawn": idx, "solves": done,
           "failures": failures}
    print(json.dumps({k: v for k, v in res.items() if k != "failures"}), f"failures={len(failures)}")
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
