#!/usr/bin/env python3
"""Benchmark of the cCG hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--arith exact|fast]
                    [--impl ours|reference] [--no-big] [--no-secondary] [--no-cpu-baseline]

Headline: config 2 (n = 16384, p = 8, diagonally dominant A, 200 fixed
iterations -- the config BASELINE.json pins to one GPU).  One
step = one full solve.  `value` = cCG iterations/s over the K timed steps with
A, b, X0 resident in HBM (CUDA events on the library's stream); `e2e` = the
same metric through the drop-in call coopcg_gpu_solve with pinned host b / X0
in and the host final X + trace out, every step; `e2e_oneshot` = the one-shot
drop-in ccg_solve(A, b, X0) with A itself uploaded from host memory every call
(what a caller of the reference's ccg_solve does once per system).
`roofline` describes Q = A.D against the north star's bound
max(8 n^2 / HBM, 2 n^2 p / FP64).  The metric is quoted "vs n, p", so the line
also carries `configs`: every other BASELINE config in both arithmetic modes
-- cfg 4 (n = 131072, p = 32, A = 137 GB on one GPU, 50 fixed iterations: the
north star's single-GPU target), cfg 3 (n = 65536, p = 16, Householder kappa =
1e6, 100 iterations), and on one GPU cfg 0 / cfg 1 (solves to 1e-10 ||b||).

--impl reference times the reference's own CPU implementation
(parallel_ccg, compiled from the unmodified reference headers into
oracle/_ref/libccgref.so) on the box's host cores, one step = one cCG
iteration of the same config, value from the reference's own per-iteration
wall times (solvers.hpp:99-105,184).  That process loads only oracle/
libraries: its inputs come from the oracle's generators (bit-identical to the
product's, tests/test_abi.py).

Multi-GPU: under torchrun (WORLD_SIZE = N > 1) every rank
opens a rank context (coopcg_gpu_create_rank): A row-block sharded, the row
exchanges are NCCL collectives enqueued by the library's own run loop.
Without torchrun, --gpus N > 1 drives N devices from this one process
(coopcg_gpu_create_multi: the Q rows are stored into every device's Q over
NVLink by the A.D kernel itself); it fails if fewer than N GPUs are visible.
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "cCG iterations/sec and A·D effective HBM GB/s (fraction of roofline) vs n, p"

# The BASELINE.json configs (paper_1204_0069_b200/configs.py holds the same
# table for the product; restated here so the reference arm never imports the
# product package).  n, p, matrix, rhs, reflectors, kappa, rel_tol, fixed_iters, seed
CFG_TABLE = {
    0: (1000, 3, "diagdom", "uniform", 0, 1.0, 1e-10, -1, 12040),
    1: (4096, 4, "householder", "normal", 8, 1e4, 1e-10, -1, 12041),
    2: (16384, 8, "diagdom", "uniform", 0, 1.0, 0.0, 200, 12042),
    3: (65536, 16, "householder", "normal", 16, 1e6, 0.0, 100, 12043),
    4: (131072, 32, "diagdom", "uniform", 0, 1.0, 0.0, 50, 12044),
}


class Cfg:
    def __init__(self, idx):
        (self.n, self.p, self.matrix, self.rhs, self.reflectors, self.kappa, self.rel_tol, self.fixed_iters,
         self.seed) = CFG_TABLE[idx]
        self.idx = idx
        self.name = f"cfg{idx}_n{self.n}_p{self.p}_{self.matrix}"


L2_BYTES = 126 * 2**20  # B200 L2


def l2_small(cfg):
    return 8.0 * cfg.n * cfg.n < 2 * L2_BYTES


def l2_note(cfg):
    a = 8.0 * cfg.n * cfg.n
    if l2_small(cfg):
        return (f"A = {a / 2**20:.0f} MB < 2x L2: L2 flushed (256 MB write) before every timed step, "
                f"outside its timing; A is L2-resident across the iterations of a step")
    return f"inputs larger than L2: A = {a / 1e9:.2f} GB streamed from HBM every iteration (L2 126 MB)"


def config_dict(cfg):
    """The `config` object, identical on both arms (the workload, not the implementation)."""
    return {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "matrix": cfg.matrix,
            "rhs": cfg.rhs, "stop": (f"fixed {cfg.fixed_iters} iterations (tol = 0)" if cfg.fixed_iters >= 0
                                     else f"||r|| <= {cfg.rel_tol:g} ||b||, max 2n iterations"),
            "x0": "column 0 = 0, columns 1.. ~ U[-1, 1] (DESIGN.md §3)", "l2": l2_note(cfg)}


def _peaks():
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            hbm = float(json.load(open(p))["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    f = json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))
    return hbm, src, f


def roofline(cfg, arith, ad_ms, n_rows=None):
    """The north star's roofline for one A.D launch: max(8 n_rows n / HBM,
    2 n_rows n p / FP64); `bound` is the larger, `frac` = roofline time /
    measured time (= achieved / peak in the bound's unit)."""
    hbm, hbm_src, f = _peaks()
    rows = cfg.n if n_rows is None else n_rows
    nbytes = 8.0 * rows * cfg.n
    flops = 2.0 * rows * cfg.n * cfg.p
    fp64 = f["dfma_tflops"]
    t_hbm = nbytes / (hbm * 1e9)
    t_f64 = flops / (fp64 * 1e12)
    gbs = nbytes / (ad_ms * 1e-3) / 1e9
    tfs = flops / (ad_ms * 1e-3) / 1e12
    r = {"ad_ms_per_launch": ad_ms, "roofline_ms": max(t_hbm, t_f64) * 1e3,
         "hbm": {"achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm, "peak_source": hbm_src},
         "fp64": {"achieved_tflops": tfs, "peak_tflops": fp64, "frac": tfs / fp64,
                  "peak_source": "profiles/fp64_peaks.json (DFMA probe, tools/probe/fp64_probe.cu)"}}
    if t_hbm >= t_f64:
        r.update({"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm})
    else:
        r.update({"bound": "fp64", "achieved": tfs, "peak": fp64, "unit": "TFLOP/s", "frac": tfs / fp64})
    if arith == "exact":
        # one DMUL + one DADD per multiply-add (the reference's separate roundings):
        # the measured DMUL+DADD issue rate (instruction lanes/s) / 2 multiply-adds/s
        tmac = f["dmul_dadd_tinstr_per_s"] / 2.0
        t_issue = rows * cfg.n * cfg.p / (tmac * 1e12) * 1e3
        r["exact_issue_ceiling"] = {"tmac_per_s": tmac, "ms": t_issue, "frac": t_issue / ad_ms,
                                    "bound_ms": max(t_issue, t_hbm * 1e3),
                                    "note": "the exact mode's own ceiling: max(HBM, DMUL+DADD issue)"}
    return r


def _traffic(cfg_name: str, arith: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        v = json.load(open(p)).get(f"{cfg_name}_{arith}", {}).get("ad_dram_bytes_per_launch")
        return float(v) if v is not None else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------
# the reference on the host (oracle/_ref): never imports the product package
# ---------------------------------------------------------------------------
def host_info(threads):
    model = platform.processor() or "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model, "threads_used": threads,
            "omp": {k: os.environ.get(k) for k in ("OMP_WAIT_POLICY", "OMP_PROC_BIND")}}


def cpu_reference_run(cfg, iters: int, serial_iters: int = 0):
    """The reference's parallel_ccg (one OpenMP thread per agent, its own
    design) on the config's inputs, `iters` iterations, and optionally its
    serial ccg_solve for `serial_iters`.  Per-iteration seconds from the
    reference's own wall times."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    os.environ.setdefault("OMP_PROC_BIND", "close")
    import pyoracle as po
    b = po.gen_rhs(cfg.n, cfg.rhs, cfg.seed)
    X0 = po.gen_starts(cfg.n, cfg.p, cfg.seed)
    tol = cfg.rel_tol * po.seq_norm(b) if cfg.fixed_iters < 0 else 0.0
    out = {}
    if po.ref_available():
        with po.RefMatrix(cfg.n) as R:
            if cfg.matrix == "diagdom":
                po.gen_diagdom_rows(cfg.n, cfg.seed, 0, cfg.n, out=R.A)
            else:
                po.gen_householder_into(cfg.n, cfg.reflectors, cfg.kappa, cfg.seed, R.A)
            tr = R.solve(b, X0, tol=tol, max_iters=iters, algo="parallel")
            out["parallel"] = ([float(w) * 1e-9 for w in tr.wall_ns], "reference", cfg.p)
            if serial_iters > 0:
                ts = R.solve(b, X0, tol=tol, max_iters=serial_iters, algo="ccg")
                out["serial"] = ([float(w) * 1e-9 for w in ts.wall_ns], "reference", 1)
    else:  # the plain-C restatement (one thread)
        A = po.gen_diagdom(cfg.n, cfg.seed) if cfg.matrix == "diagdom" else \
            po.gen_householder(cfg.n, cfg.reflectors, cfg.kappa, cfg.seed)
        tr = po.oracle_ccg(A, b, X0, tol=tol, max_iters=iters)
        out["parallel"] = ([float(w) * 1e-9 for w in tr.wall_ns], "port", 1)
    return out


def run_reference_arm(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    total = args.warmup + args.steps
    runs = cpu_reference_run(cfg, total, serial_iters=(args.serial_iters if cfg.n <= 16384 else 0))
    walls, kind, cores = runs["parallel"]
    timed = walls[args.warmup:args.warmup + args.steps]
    if len(timed) < args.steps:
        print(json.dumps({"impl": "reference", "unavailable": "reference solve stopped early"}))
        return 0
    secs = sum(timed)
    value = len(timed) / secs
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": value, "unit": "iterations/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / len(timed) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 generators, DESIGN.md §3)",
        "config": config_dict(cfg),
        "step": "one cCG iteration of the config (bounded sample of the solve)",
        "solver": "parallel_ccg (reference headers compiled unmodified, OpenMP, one thread per agent: "
                  "parallel.hpp:76-111 requires workers == p)",
        "host": host_info(cores),
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": kind,
                         "sample": f"{args.steps} timed iterations after {args.warmup} warm-up of {cfg.name}"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if "serial" in runs:
        sw = runs["serial"][0]
        line["serial_ccg_solve"] = {"s_per_iteration": sum(sw) / len(sw), "iterations": len(sw),
                                    "value": len(sw) / sum(sw), "unit": "iterations/s", "threads": 1}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def _measure(m, torch, cfg, args, arith, steps, warmup, ctx_kw, e2e=True, clock_dev=0, barrier=None,
             reduce_max=None):
    """Resident-A solves timed with CUDA events on the library stream (shard 0's
    for a multi-device handle; the max over ranks for rank contexts), then the
    drop-in e2e call with pinned host buffers."""
    import ctypes as C
    import numpy as np
    from paper_1204_0069_b200 import _capi
    from paper_1204_0069_b200.configs import CONFIGS, make_problem_on_device

    pcfg = CONFIGS[cfg.idx]
    if callable(ctx_kw.get("nccl")):  # rank contexts: a fresh NCCL id per communicator
        ctx_kw = dict(ctx_kw, nccl=ctx_kw["nccl"]())
    ctx = m.GpuContext(cfg.n, cfg.p, arith=arith, **ctx_kw)
    b, X0, opts = make_problem_on_device(ctx, pcfg)
    ctx.upload(b, X0)
    dev, row0, row1 = ctx.shards()[0]  # shard 0 (its stream carries the events; its rows the A.D timing)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    for _ in range(warmup):
        ctx.run_raw(opts)
    torch.cuda.synchronize(dev)
    flush = (torch.empty(256 * 2**20 // 8, dtype=torch.float64, device=f"cuda:{dev}") if l2_small(cfg) else None)

    def flush_l2():
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)

    iters_total = mv_ms = 0.0
    mv_n = launches = checks = 0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if barrier:
        barrier()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(clock_dev) if clock_dev is not None else contextlib.nullcontext()
    with sampler:
        for e0, e1 in evs:
            flush_l2()
            e0.record(stream)
            its, ch = ctx.run_raw(opts)
            e1.record(stream)
            iters_total += its
            checks += ch
            tm = ctx.timing()
            mv_ms += tm["matvec_ms_total"]
            mv_n += tm["matvec_launches"]
            launches += tm["kernel_launches"]
        torch.cuda.synchronize(dev)
    elapsed_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    if barrier:
        barrier()
    if reduce_max:
        elapsed_ms = reduce_max(elapsed_ms)
    res = {"value": iters_total / (elapsed_ms * 1e-3), "ms_per_step": elapsed_ms / steps,
           "iterations_per_step": int(iters_total) // max(steps, 1), "exact_rank_fallbacks": checks,
           "gpu_launches": launches, "steps": steps, "warmup": warmup,
           "clocks": sampler.summary() if hasattr(sampler, "summary") else None}
    if mv_n == 0:
        raise RuntimeError("no A.D launch was timed (COOPCG_MV_EVERY=0?); the roofline needs sampled launches")
    res["roofline"] = roofline(cfg, arith, mv_ms / mv_n, row1 - row0)
    res["roofline"]["ad_launches_timed"] = mv_n
    res["roofline"]["traffic"] = _traffic(cfg.name, arith)
    res["roofline"]["kernel"] = ("ad_exact_pipe_kernel (p <= 16) / ad_exact_rpt_kernel (p = 32): Q = A.D, "
                                 "separate DMUL/DADD (DESIGN.md §5)" if arith == "exact"
                                 else "ad_fast_kernel: Q = A.D on DMMA m8n8k4 (DESIGN.md §5)")

    if e2e:
        n, p = cfg.n, cfg.p
        bh = torch.from_numpy(b).pin_memory()
        X0c = torch.from_numpy(np.ascontiguousarray(X0.T)).pin_memory()
        fx = torch.empty((p, n), dtype=torch.float64).pin_memory()
        L = _capi.lib()
        cap = max(opts.max_iters if opts.max_iters >= 0 else 2 * n, 1)
        norms = torch.empty((cap, p), dtype=torch.float64).pin_memory()
        tr = _capi.coopcg_trace()
        tr.capacity = cap
        tr.residual_norms = C.cast(norms.data_ptr(), C.POINTER(C.c_double))
        tr.final_x = C.cast(fx.data_ptr(), C.POINTER(C.c_double))
        co = opts.to_c()

        def e2e_once():
            rc = L.coopcg_gpu_solve(ctx._h, C.c_void_p(bh.data_ptr()), C.c_void_p(X0c.data_ptr()),
                                    C.byref(co), C.byref(tr))
            if rc != 0:
                raise RuntimeError(f"coopcg_gpu_solve failed: {rc}")
            return tr.iterations

        e2e_once()
        torch.cuda.synchronize(dev)
        e2e_iters, e2e_s = 0, 0.0
        with (ClockSampler(clock_dev) if clock_dev is not None else contextlib.nullcontext()):
            for _ in range(steps):
                flush_l2()
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                e2e_iters += e2e_once()  # returns after the final X and trace are on the host
                e2e_s += time.perf_counter() - t0
        if reduce_max:
            e2e_s = reduce_max(e2e_s)
        res["e2e"] = {"value": e2e_iters / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": (n + n * p) * 8,
                      "d2h_bytes_per_step": (n * p + tr.iterations * p) * 8,
                      "call": "coopcg_gpu_solve (resident A; pinned b, X0 in; final X + residual history out)"}
    ctx.close()
    return res, (b, X0, opts)


def _oneshot_e2e(m, torch, cfg, arith, steps, dev):
    """The one-shot drop-in ccg_solve(A, b, X0) (the call a user of the
    reference's ccg_solve makes): context creation, A uploaded from (pageable)
    host memory, solve, trace + X back, context destroyed -- every step."""
    from paper_1204_0069_b200.configs import CONFIGS, make_problem_on_device
    pcfg = CONFIGS[cfg.idx]
    with m.GpuContext(cfg.n, cfg.p, device=dev, arith=arith) as ctx:
        b, X0, opts = make_problem_on_device(ctx, pcfg)
        A = ctx.get_A()
    gpu = m.GpuOptions(device=dev, arith=arith)
    m.ccg_solve(A, b, X0, opts, gpu)  # warm
    its, secs = 0, 0.0
    for _ in range(steps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        t = m.ccg_solve(A, b, X0, opts, gpu)
        secs += time.perf_counter() - t0
        its += t.iteration_count()
    return {"value": its / secs, "unit": "iterations/s", "s_per_call": secs / steps,
            "h2d_bytes_per_step": 8 * (cfg.n * cfg.n + cfg.n + cfg.n * cfg.p),
            "d2h_bytes_per_step": 8 * (cfg.n * cfg.p + t.iteration_count() * cfg.p),
            "call": "paper_1204_0069_b200.ccg_solve(A, b, X0) = coopcg::gpu_ccg: create, set_A (host A), "
                    "solve, destroy"}


def run_ours(args, cfg):
    import torch
    import paper_1204_0069_b200 as m

    ws, rank, local = _dist()
    barrier = reduce_max = None
    if ws > 1 or args.rank_path:
        if args.gpus not in (1, ws):
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")  # control plane only; the row exchanges are NCCL inside the library
        def fresh_id():
            uid = [m.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            return (ws, rank, uid[0])
        ctx_kw = {"device": local, "nccl": fresh_id}
        barrier = dist.barrier

        def reduce_max(x):
            t = torch.tensor([float(x)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        n_gpus = ws
        parallelism = (f"row-block sharded A over {ws} ranks (one process per GPU); NCCL all-gather of the Q "
                       "rows (+ R / S rows) enqueued by the library's run loop (coopcg_gpu_create_rank)")
        clock_dev = local if rank == 0 else None
    else:
        n_gpus = args.gpus
        if n_gpus > 1:
            if torch.cuda.device_count() < n_gpus:
                raise SystemExit(f"bench.py --gpus {n_gpus}: only {torch.cuda.device_count()} GPU(s) visible")
            ctx_kw = {"devices": list(range(n_gpus))}
            parallelism = (f"row-block sharded A over {n_gpus} GPUs driven by one process "
                           "(coopcg_gpu_create_multi): the A.D kernel stores its Q rows into every GPU's Q over "
                           "NVLink peer memory, cross-stream event barrier")
        else:
            ctx_kw = {"device": args.device}
            parallelism = "single GPU"
        clock_dev = args.device
        torch.cuda.set_device(args.device)

    main, (b, X0, opts) = _measure(m, torch, cfg, args, args.arith, args.steps, args.warmup, ctx_kw,
                                   clock_dev=clock_dev, barrier=barrier, reduce_max=reduce_max)
    line = {
        "metric": BASELINE_METRIC, "value": main["value"], "unit": "iterations/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 generators, DESIGN.md §3; A generated on device)",
        "config": config_dict(cfg),
        "arith": args.arith,
        "step": f"one full solve ({main['iterations_per_step']} iterations + setup + true-residual finalize)",
        "parity": ("exact: bit-identical to the reference's parallel_ccg at this config "
                   "(tests/test_gpu_full_configs.py, all 200 iterations)" if args.arith == "exact" else
                   "fast: X within 1e-8, history within 1e-8 before k_div (tests/test_gpu_full_configs.py)"),
        "parallelism": parallelism,
        "exact_rank_fallbacks": main["exact_rank_fallbacks"],
        "roofline": main["roofline"], "e2e": main["e2e"], "gpu_launches": main["gpu_launches"],
        "clocks": main["clocks"],
    }
    big_ok = ws == 1 and n_gpus == 1 and not args.rank_path
    if not args.no_secondary:
        other = "fast" if args.arith == "exact" else "exact"
        r2, _ = _measure(m, torch, cfg, args, other, args.steps, args.warmup, ctx_kw, clock_dev=clock_dev,
                         barrier=barrier, reduce_max=reduce_max)
        line[other] = {k: r2[k] for k in ("value", "ms_per_step", "roofline", "e2e", "gpu_launches", "clocks")}
        line[other]["unit"] = "iterations/s"
    if big_ok and not args.no_oneshot:
        line["e2e_oneshot"] = _oneshot_e2e(m, torch, cfg, args.arith, max(1, min(args.steps, 3)), args.device)
    if not args.no_big:
        # The metric is quoted "vs n, p": the same line carries every other BASELINE
        # config, timed the same way in both modes -- the north star's single-GPU
        # target (cfg 4: n = 131072, p = 32, A = 137 GB) and cfg 3 (n = 65536) with
        # --big-steps timed solves each, the small configs (cfg 0 / 1) with --steps.
        line["configs"] = {}
        for idx in ((0, 1, 3, 4) if big_ok else (3, 4)):  # multi-GPU runs: the sharded configs only
            if idx == cfg.idx:
                continue
            other_cfg = Cfg(idx)
            obj = {"config": config_dict(other_cfg), "modes": {}}
            for arith in ("exact", "fast"):
                r, _ = _measure(m, torch, other_cfg, args, arith, args.big_steps if idx >= 3 else args.steps,
                                args.warmup, ctx_kw, e2e=True, clock_dev=clock_dev, barrier=barrier,
                                reduce_max=reduce_max)
                r["unit"] = "iterations/s"
                obj["modes"][arith] = r
            if idx >= 3:
                obj["cpu_reference"] = (
                    "not run by bench.py (a 34 / 137 GB host copy of A; 4 / 42 s per iteration with the "
                    "reference's one thread per agent on 16 cores): measured per iteration by "
                    "tests/test_gpu_full_configs.py (profiles/r02_full_config_parity.json)")
            line["configs"][f"cfg{idx}"] = obj
    if not args.no_cpu_baseline and rank == 0:
        runs = cpu_reference_run(cfg, args.cpu_iters)
        walls, kind, cores = runs["parallel"]
        secs = sum(walls)
        line["cpu_baseline"] = {"value": len(walls) / secs if secs > 0 else None, "unit": "iterations/s",
                                "cores": cores, "kind": kind, "host": host_info(cores),
                                "sample": f"{len(walls)} iterations of {cfg.name} (parallel_ccg, one thread per "
                                          "agent; the reference's per-iteration wall times)"}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1 or args.rank_path:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--arith", default="exact", choices=["exact", "fast"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--device", type=int, default=int(os.environ.get("LOCAL_RANK", "0")))
    ap.add_argument("--cpu-iters", type=int, default=8)
    ap.add_argument("--serial-iters", type=int, default=3, help="reference arm: serial ccg_solve sample (cfg <= 2)")
    ap.add_argument("--big-steps", type=int, default=2, help="timed solves of the cfg3 / cfg4 objects")
    ap.add_argument("--no-big", action="store_true", help="skip the other BASELINE configs (the `configs` object)")
    ap.add_argument("--no-oneshot", action="store_true", help="skip the one-shot e2e (A uploaded every call)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the other arithmetic mode")
    ap.add_argument("--rank-path", action="store_true",
                    help="(testing) take the one-process-per-GPU rank-context path even with one rank under torchrun")
    args = ap.parse_args()
    cfg = Cfg(args.config)
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
