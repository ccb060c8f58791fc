#!/usr/bin/env python3
"""Benchmark of the cCG hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--arith exact|fast]
                    [--impl ours|reference]

One step = one full solve of the selected BASELINE config (default: config 2,
n=16384, p=8, diagonally dominant A, 200 fixed iterations -- the largest
config BASELINE.json pins to one GPU; DESIGN.md §6 says why).  `value` is
cCG iterations/s over the K timed steps with A, b, X0 resident in HBM, timed
with CUDA events on the library's own stream; `e2e` is the same metric
through the drop-in call (coopcg_gpu_solve) with pinned host buffers, the
host->device copy of b/X0 and the device->host copy of X/trace inside the
timed region.  `roofline` describes the dominant kernel (Q = A.D).

--impl reference times the reference's own CPU implementation
(parallel_ccg, compiled from the reference headers into oracle/_ref) on the
host cores, one step = one cCG iteration of the same config, value from the
reference's own per-iteration wall times (solvers.hpp:99-105,184).

Multi-GPU (torchrun, N>1): A is row-block sharded across ranks
(paper_1204_0069_b200.sharded); value = iterations/s of the sharded solve.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "cCG iterations/sec and A·D effective HBM GB/s (fraction of roofline) vs n, p"


def _peaks():
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            hbm = float(json.load(open(p))["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    # FP64 peak: measured with tools/probe/fp64_probe (DFMA 36.0, DMMA 36.9 TF/s).
    fp64 = 36.0
    return hbm, src, fp64


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

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
        self.out = ""
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
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_run(cfg, iters: int, threads_note: str = ""):
    """The reference's parallel_ccg (oracle/_ref) on the config's inputs,
    `iters` iterations.  Returns (iterations/s, per-iteration seconds list, kind, cores)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle as po
    from paper_1204_0069_b200.configs import host_inputs, seq_norm
    if cfg.matrix == "diagdom":
        A = po.gen_diagdom(cfg.n, cfg.seed)
    else:
        A = po.gen_householder(cfg.n, cfg.reflectors, cfg.kappa, cfg.seed)
    b, X0 = host_inputs(cfg)
    tol = cfg.rel_tol * seq_norm(b) if cfg.fixed_iters < 0 else 0.0
    os.environ.setdefault("OMP_WAIT_POLICY", "passive")
    os.environ.setdefault("OMP_PROC_BIND", "close")
    if po.ref_available():
        tr = po.ref_solve(A, b, X0, tol=tol, max_iters=iters, algo="parallel")
        kind, cores = "reference", cfg.p
    else:
        tr = po.oracle_ccg(A, b, X0, tol=tol, max_iters=iters)
        kind, cores = "port", 1
    walls = [float(w) * 1e-9 for w in tr.wall_ns]
    return walls, kind, cores


def run_reference_arm(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    total = args.warmup + args.steps
    walls, kind, cores = cpu_reference_run(cfg, total)
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
        "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "step": "one cCG iteration",
                   "solver": "parallel_ccg (reference, OpenMP, one thread per agent)"},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": kind,
                         "sample": f"{args.steps} timed iterations after {args.warmup} warm-up of {cfg.name}"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def _profile_traffic(cfg_name: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            v = d.get(cfg_name, {}).get("ad_dram_bytes_per_launch")
            return float(v) if v is not None else None
        except Exception:
            return None
    return None


L2_BYTES = 126 * 2**20  # B200 L2 (nvidia-smi / MEASURED_PEAKS box)


def l2_small(cfg):
    return 8.0 * cfg.n * cfg.n < 2 * L2_BYTES


def l2_note(cfg):
    a = 8.0 * cfg.n * cfg.n
    if l2_small(cfg):
        return (f"A = {a / 2**20:.0f} MB < 2x L2: L2 flushed (256 MB write) before every timed step, "
                f"outside its timing; A is L2-resident across the iterations of a step")
    return f"inputs larger than L2: A = {a / 1e9:.2f} GB streamed from HBM every iteration (L2 126 MB)"


def l2_flush_buffer(torch, cfg, dev):
    if not l2_small(cfg):
        return None
    return torch.empty(256 * 2**20 // 8, dtype=torch.float64, device=f"cuda:{dev}")


def _measure(m, torch, cfg, args, arith, dev):
    """K timed solves (inputs resident) + K e2e solves through the drop-in call."""
    import ctypes as C
    import numpy as np
    from paper_1204_0069_b200 import _capi
    from paper_1204_0069_b200.configs import make_problem_on_device

    ctx = m.GpuContext(cfg.n, cfg.p, device=dev, arith=arith)
    b, X0, opts = make_problem_on_device(ctx, cfg)
    ctx.upload(b, X0)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    for _ in range(args.warmup):
        ctx.run(opts, want_x=False)
    torch.cuda.synchronize()
    iters_total = 0
    mv_ms = 0.0
    mv_n = 0
    launches = 0
    exact_rank_checks = 0
    # L2 rule: A larger than L2 streams from HBM every iteration; otherwise L2 is
    # flushed (a 256 MB write on the library stream) before every timed step,
    # outside its event pair (A then stays L2-resident across the iterations of
    # the step, as it does for the reference on its host caches).
    flush = l2_flush_buffer(torch, cfg, dev)

    def flush_l2():
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for e0, e1 in evs:
            flush_l2()
            e0.record(stream)
            its, checks = ctx.run_raw(opts)  # the C solve call only (no Python trace assembly)
            e1.record(stream)
            iters_total += its
            exact_rank_checks += checks
            tm = ctx.timing()
            mv_ms += tm["matvec_ms_total"]
            mv_n += tm["matvec_launches"]
            launches += tm["kernel_launches"]
        torch.cuda.synchronize()
    elapsed_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)

    # e2e: the drop-in call (coopcg_gpu_solve) with pinned host buffers
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

    e2e_once()  # warm (pinned registration etc.)
    torch.cuda.synchronize()
    e2e_iters = 0
    e2e_s = 0.0
    # same host load as the timed loop (the clock sampler thread runs in both)
    with ClockSampler(dev):
        for _ in range(args.steps):
            flush_l2()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_iters += e2e_once()  # returns after the final X and trace are on the host
            e2e_s += time.perf_counter() - t0
    h2d = (n + n * p) * 8
    d2h = (n * p + tr.iterations * p) * 8

    hbm_peak, peak_src, fp64_peak = _peaks()
    if mv_n == 0:
        raise RuntimeError("no A.D launch was timed (COOPCG_MV_EVERY=0?); the roofline needs sampled launches")
    ad_ms = mv_ms / mv_n
    ad_bytes = 8.0 * cfg.n * cfg.n
    ad_flops = 2.0 * cfg.n * cfg.n * cfg.p
    achieved = ad_bytes / (ad_ms * 1e-3) / 1e9
    ctx.close()
    return {
        "value": iters_total / (elapsed_ms * 1e-3),
        "ms_per_step": elapsed_ms / args.steps,
        "iterations_per_step": iters_total // max(args.steps, 1),
        "exact_rank_checks": exact_rank_checks,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": _profile_traffic(f"{cfg.name}_{arith}"),
                     "kernel": ("exact Q = A.D (ad_exact_pipe_kernel at the BASELINE configs with p <= 16, "
                                "ad_exact_rpt_kernel at p = 32; DESIGN.md §5)") if arith == "exact"
                     else "ad_fast_kernel (Q = A.D, DMMA)",
                     "ad_ms_per_launch": ad_ms, "ad_launches_timed": mv_n, "peak_source": peak_src,
                     "fp64": {"achieved_tflops": ad_flops / (ad_ms * 1e-3) / 1e12, "peak_tflops": fp64_peak,
                              "peak_source": "measured DFMA/DMMA probe (tools/probe/fp64_probe.cu)",
                              # exact mode keeps both roundings: one DMUL + one DADD per multiply-add,
                              # 18.2 T FP64 instructions/s measured = 18.2 TF/s-equivalent
                              "exact_issue_ceiling_tflops": 18.2 if arith == "exact" else None},
                     "roofline_ms": max(ad_bytes / (hbm_peak * 1e9), ad_flops / (fp64_peak * 1e12)) * 1e3},
        "e2e": {"value": e2e_iters / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
    }


def run_ours(args, cfg):
    import torch
    import paper_1204_0069_b200 as m

    ws, rank, local = _dist()
    if ws > 1 or args.sharded_path:
        from paper_1204_0069_b200 import sharded
        return sharded.bench_main(args, cfg, BASELINE_METRIC, clock_sampler=ClockSampler, peaks=_peaks)
    dev = args.device
    torch.cuda.set_device(dev)
    main_arith = args.arith
    res = _measure(m, torch, cfg, args, main_arith, dev)
    line = {
        "metric": BASELINE_METRIC, "value": res["value"], "unit": "iterations/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 generators, DESIGN.md §3; A generated on device)",
        "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "matrix": cfg.matrix,
                   "iterations_per_step": res["iterations_per_step"], "arith": main_arith,
                   "parity": ("bit-identical to the reference ccg_solve (tests/test_gpu_parity.py)"
                              if main_arith == "exact" else
                              "X within 1e-8, pre-floor history within 1e-8 (tests/test_gpu_fast.py)"),
                   "step": "one full solve (setup + iterations + true-residual finalize)",
                   "l2": l2_note(cfg),
                   "parallelism": "single GPU", "exact_rank_fallbacks": res["exact_rank_checks"]},
        "roofline": res["roofline"],
        "e2e": res["e2e"],
        "gpu_launches": res["gpu_launches"],
        "clocks": res["clocks"],
    }
    if not args.no_secondary:
        other = "fast" if main_arith == "exact" else "exact"
        r2 = _measure(m, torch, cfg, args, other, dev)
        line[other] = {"value": r2["value"], "unit": "iterations/s", "ms_per_step": r2["ms_per_step"],
                       "roofline": r2["roofline"], "e2e": r2["e2e"], "gpu_launches": r2["gpu_launches"],
                       "clocks": r2["clocks"],
                       "parity": ("X within 1e-8, pre-floor history within 1e-8, +-2 iterations "
                                  "(tests/test_gpu_fast.py); not bit-identical by design"
                                  if other == "fast" else "bit-identical")}
    if not args.no_cpu_baseline:
        walls, kind, cores = cpu_reference_run(cfg, args.cpu_iters)
        secs = sum(walls)
        line["cpu_baseline"] = {"value": len(walls) / secs if secs > 0 else None, "unit": "iterations/s",
                                "cores": cores, "kind": kind,
                                "sample": f"{len(walls)} iterations of {cfg.name} (parallel_ccg, "
                                          "reference per-iteration wall times)"}
    print(json.dumps(line))
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the other arithmetic mode")
    ap.add_argument("--sharded-path", action="store_true",
                    help="(testing) drive the row-sharded orchestrator even with one rank under torchrun")
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1: exchange Q through peer memory (CUDA IPC push from the A.D kernel) instead of "
                         "an NCCL all-gather")
    args = ap.parse_args()
    from paper_1204_0069_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
