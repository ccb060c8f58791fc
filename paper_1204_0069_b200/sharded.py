"""Row-sharded multi-GPU cCG.

Rank g of G owns rows [row0, row1) of A (evenly split, ceil(n/G) rows per
rank).  Every n x p block (X, R, D, Q) and the p x p state are replicated;
per iteration each rank computes its rows of Q = A_g D, one all-gather of Q
makes Q complete everywhere, and every rank then runs the identical rest of
the iteration.  Residual recomputations (every 50th iteration,
solvers.hpp:33-35) add one all-gather of the new R rows; setup and the final
true residual add one each.  In exact mode the result is bit-identical to a
single-GPU (and to the reference) solve for any G: each row's A-chain is
local and every other value is computed identically on every rank.

The orchestrator is written against a small "engine" protocol so that the
same code drives the CUDA library (GpuShardEngine, NCCL) and the oracle-backed
CPU engine of tests/test_sharded_gloo.py (gloo):

    engine.row0, engine.row1, engine.n, engine.P, engine.max_iters
    engine.begin(opts); engine.phase(ph, k); engine.recompute_at(k) -> bool
    engine.block(which, k) -> torch tensor (n x P) view of that block
    engine.state() -> (stop, iterations); engine.end() -> SolveTrace
    engine.mccg_resume() -> k to resume from after an mccg restriction, or -1
    engine.collective_stream() -> context manager ordering collectives with
                                  the engine's stream

Peer mode (GpuShardEngine.enable_peers + PeerQExchange): the Q rows are
pushed into every rank's Q by the kernel that computes them (CUDA IPC
mappings; one fused compute + exchange step), and the per-iteration Q
"all-gather" reduces to a stream-ordered barrier.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import json
import os
import time
from typing import Optional

import numpy as np

from . import _capi
from .solver import GpuContext, SolveOptions, _check, _dp

PH_SETUP_LOCAL, PH_SETUP_REST, PH_ITER_LOCAL, PH_ITER_MID, PH_ITER_REST, PH_FINAL_LOCAL, PH_FINAL_REST, PH_MCCG_SETUP = range(8)
BLOCK_X, BLOCK_R, BLOCK_D, BLOCK_Q, BLOCK_S, BLOCK_W = range(6)


def row_split(n: int, world: int, rank: int):
    """Even row blocks: ceil(n / world) rows per rank (the last may be short)."""
    per = (n + world - 1) // world
    r0 = min(n, rank * per)
    return r0, min(n, r0 + per), per


class RowExchange:
    """All-gather of row blocks of an n x P block over torch.distributed."""

    def __init__(self, n: int, P: int, world: int, rank: int, group=None):
        import torch
        self.n, self.P, self.world, self.rank, self.group = n, P, world, rank, group
        self.r0, self.r1, self.per = row_split(n, world, rank)
        self.even = self.per * world == n
        self._stage = {}
        self._torch = torch

    def allgather(self, block) -> None:
        """block: (n, P) tensor whose rows [r0, r1) are this rank's; fills the rest."""
        torch = self._torch
        import torch.distributed as dist
        if self.world == 1:
            return
        if self.even:
            dist.all_gather_into_tensor(block, block[self.r0:self.r1], group=self.group)
            return
        key = (block.device, block.dtype)
        if key not in self._stage:
            self._stage[key] = (torch.zeros((self.per * self.world, self.P), dtype=block.dtype, device=block.device),
                                torch.zeros((self.per, self.P), dtype=block.dtype, device=block.device))
        out, inp = self._stage[key]
        inp.zero_()
        inp[: self.r1 - self.r0].copy_(block[self.r0:self.r1])
        dist.all_gather_into_tensor(out, inp, group=self.group)
        block.copy_(out[: self.n])

    def allgather_q(self, block) -> None:
        """The per-iteration exchange of Q (an all-gather here)."""
        self.allgather(block)


class PeerQExchange(RowExchange):
    """Peer mode: Q rows arrive through the peer push of the producing kernel;
    the Q exchange is only a barrier ordered after it on every rank (a
    one-element all-reduce on the context stream with NCCL; a stream sync plus
    a host barrier with gloo).  R and S are still all-gathered."""

    def __init__(self, n: int, P: int, world: int, rank: int, group=None, device: int = 0):
        super().__init__(n, P, world, rank, group)
        import torch.distributed as dist
        self._nccl = dist.get_backend(group) == "nccl"
        self._flag = self._torch.zeros(1, dtype=self._torch.float64, device=f"cuda:{device}")

    def allgather_q(self, block) -> None:
        torch = self._torch
        import torch.distributed as dist
        if self.world == 1:
            return
        if self._nccl:
            dist.all_reduce(self._flag, group=self.group)  # stream-ordered after this rank's push
        else:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)


def gen_householder_sharded(engine, exchange_w: RowExchange, seed: int, m: int, kappa: float) -> None:
    """The Householder generator on row-sharded contexts: each
    rank computes its rows of w = M v, the ranks all-gather w (an n x 1
    RowExchange), and each rank updates its own rows of M with the scalars
    every rank forms identically from the full vectors
    (include/coopcg_gpu.h, coopcg_gpu_gen_householder_*)."""
    L = _capi.lib()
    h = engine.ctx._h
    _check(h, L.coopcg_gpu_gen_householder_begin(h, seed, m, kappa))
    w = engine.vector(BLOCK_W)
    for r in range(m - 1, -1, -1):
        _check(h, L.coopcg_gpu_gen_householder_local(h, r))
        with engine.collective_stream():
            exchange_w.allgather(w)
        _check(h, L.coopcg_gpu_gen_householder_rest(h, r))
    _check(h, L.coopcg_gpu_gen_householder_end(h))


def solve_sharded(engine, exchange: RowExchange, opts: SolveOptions, poll_every: int = 8):
    """Drive one sharded solve (the phase protocol of include/coopcg_gpu.h)."""
    engine.begin(opts)
    engine.phase(PH_SETUP_LOCAL, 0)
    with engine.collective_stream():
        exchange.allgather(engine.block(BLOCK_R, 0))
    engine.phase(PH_SETUP_REST, 0)
    mccg = opts.algo == "mccg"
    if mccg:
        engine.phase(PH_MCCG_SETUP, 0)
    stop, _ = engine.state()
    k = 0
    while True:
        while not stop and k < engine.max_iters:
            engine.phase(PH_ITER_LOCAL, k)
            with engine.collective_stream():
                exchange.allgather_q(engine.block(BLOCK_Q, k))
            engine.phase(PH_ITER_MID, k)
            if engine.recompute_at(k):
                with engine.collective_stream():
                    exchange.allgather(engine.block(BLOCK_R, k))
            engine.phase(PH_ITER_REST, k)
            k += 1
            # Every rank polls at the same k and, computing identical values,
            # sees the same stop flag: the collectives stay matched.
            if k % poll_every == 0 or k >= engine.max_iters:
                stop, _ = engine.state()
        # mccg: a rank drop paused every rank at the same iteration; each
        # restricts its replicated blocks identically and all resume together
        # (the iterations enqueued after the pause were no-ops)
        if not (mccg and stop):
            break
        k = engine.mccg_resume()
        if k < 0:
            break
        stop = False
    engine.phase(PH_FINAL_LOCAL, 0)
    with engine.collective_stream():
        exchange.allgather(engine.block(BLOCK_S, 0))
    engine.phase(PH_FINAL_REST, 0)
    return engine.end()


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can view library device memory."""

    def __init__(self, ptr: int, shape, device: int):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class GpuShardEngine:
    """The CUDA library context for one row block (one GPU per rank)."""

    def __init__(self, n: int, p: int, rank: int, world: int, device: int, arith: str = "exact"):
        import torch
        self.n, self.p = n, p
        self.row0, self.row1, _ = row_split(n, world, rank)
        self.ctx = GpuContext(n, p, device=device, arith=arith, row_begin=self.row0, row_end=self.row1)
        self.device = device
        self._torch = torch
        self._stream = torch.cuda.ExternalStream(self.ctx.stream_handle(), device=device)
        ptr = C.c_void_p()
        ld = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_block(self.ctx._h, BLOCK_X, 0, C.byref(ptr), C.byref(ld)))
        self.P = ld.value
        self._views = {}
        self.max_iters = 0
        self.opts = None

    def enable_peers(self, group=None):
        """Peer-memory Q exchange: share this context's Q buffers (CUDA IPC) with
        every rank of `group` and map theirs (include/coopcg_gpu.h)."""
        import torch.distributed as dist
        own = (C.c_char * 128)()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_ipc_handles(self.ctx._h, own))
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        allh = [None] * world
        dist.all_gather_object(allh, bytes(own), group=group)
        buf = (C.c_char * (128 * world)).from_buffer_copy(b"".join(allh))
        _check(self.ctx._h, _capi.lib().coopcg_gpu_set_peers(self.ctx._h, world, rank, buf))
        self._views.clear()

    def block(self, which: int, k: int):
        ptr = C.c_void_p()
        ld = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_block(self.ctx._h, which, k, C.byref(ptr), C.byref(ld)))
        key = ptr.value
        if key not in self._views:
            self._views[key] = self._torch.as_tensor(_CudaArray(ptr.value, (self.n, self.P), self.device),
                                                     device=f"cuda:{self.device}")
        return self._views[key]

    def vector(self, which: int):
        """(n, 1) torch view of a device vector of the context (COOPCG_BLOCK_W)."""
        ptr = C.c_void_p()
        ld = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_block(self.ctx._h, which, 0, C.byref(ptr), C.byref(ld)))
        return self._torch.as_tensor(_CudaArray(ptr.value, (self.n, 1), self.device), device=f"cuda:{self.device}")

    def collective_stream(self):
        return self._torch.cuda.stream(self._stream)

    def begin(self, opts: SolveOptions):
        self.opts = opts
        self.max_iters = opts.max_iters if opts.max_iters >= 0 else 2 * self.n
        co = opts.to_c()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_begin(self.ctx._h, C.byref(co)))

    def phase(self, ph: int, k: int):
        _check(self.ctx._h, _capi.lib().coopcg_gpu_phase(self.ctx._h, ph, k))

    def recompute_at(self, k: int) -> bool:
        return bool(_capi.lib().coopcg_gpu_recompute_at(self.ctx._h, k))

    def mccg_resume(self) -> int:
        nk = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_mccg_resume(self.ctx._h, C.byref(nk)))
        return nk.value

    def state(self):
        stop = C.c_int()
        it = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_state(self.ctx._h, C.byref(stop), C.byref(it)))
        return bool(stop.value), it.value

    def end(self, want_x: bool = True):
        n, p = self.n, self.p
        cap = max(self.max_iters, 1)
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
        _check(self.ctx._h, _capi.lib().coopcg_gpu_end(self.ctx._h, C.byref(tr)))
        return self.ctx._make_trace(tr, norms, minres, wall, init, fres, fx, self.opts, act)

    def close(self):
        self.ctx.close()


def bench_main(args, cfg, metric: str, clock_sampler=None, peaks=None) -> int:
    """bench.py under torchrun: row-sharded solve of `cfg` on WORLD_SIZE GPUs.

    value: iterations / max over ranks of the summed CUDA-event time of the
    timed solves (inputs resident); e2e: b and X0 uploaded from host and the
    final X + trace downloaded every step, wall clock, max over ranks.
    --p2p: the peer-memory Q exchange instead of the NCCL all-gather of Q."""
    import torch
    import torch.distributed as dist
    from .configs import host_inputs, solve_options
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    p2p = bool(getattr(args, "p2p", False))
    eng = GpuShardEngine(cfg.n, cfg.p, rank, world, local, arith=args.arith)
    if cfg.matrix == "householder":
        gen_householder_sharded(eng, RowExchange(cfg.n, 1, world, rank), cfg.seed, cfg.reflectors, cfg.kappa)
    else:
        eng.ctx.gen_A(cfg.matrix, cfg.seed, cfg.reflectors, cfg.kappa)
    b, X0 = host_inputs(cfg)
    opts = solve_options(cfg, b)
    eng.ctx.upload(b, X0)
    if p2p:
        eng.enable_peers()
        ex = PeerQExchange(cfg.n, eng.P, world, rank, None, local)
    else:
        ex = RowExchange(cfg.n, eng.P, world, rank)
    for _ in range(args.warmup):
        solve_sharded(eng, ex, opts)
    torch.cuda.synchronize()
    dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    iters = 0
    mv_ms, mv_n, launches = 0.0, 0, 0
    sampler = clock_sampler(local) if (clock_sampler is not None and rank == 0) else contextlib.nullcontext()
    with sampler:
        for e0, e1 in evs:
            e0.record(eng._stream)
            t = solve_sharded(eng, ex, opts)
            e1.record(eng._stream)
            iters += t.iteration_count()
            tm = eng.ctx.timing()
            mv_ms += tm["matvec_ms_total"]
            mv_n += tm["matvec_launches"]
            launches += tm["kernel_launches"]
        torch.cuda.synchronize()
    ms = torch.tensor([sum(e0.elapsed_time(e1) for e0, e1 in evs)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # e2e: host inputs up, final X + trace down, every step
    dist.barrier()
    e2e_iters, t0 = 0, time.perf_counter()
    for _ in range(args.steps):
        eng.ctx.upload(b, X0)
        e2e_iters += solve_sharded(eng, ex, opts).iteration_count()
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], device=f"cuda:{local}")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        secs = float(ms.item()) * 1e-3
        hbm_peak, peak_src, fp64_peak = peaks() if peaks is not None else (6541.5, "fallback", 36.0)
        n_loc = eng.row1 - eng.row0
        ad_ms = mv_ms / max(mv_n, 1)
        ad_bytes = 8.0 * cfg.n * n_loc
        achieved = ad_bytes / (ad_ms * 1e-3) / 1e9 if mv_n else None
        line = {
            "metric": metric, "value": iters / secs, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64 generators, DESIGN.md §3)",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "arith": args.arith,
                       "parallelism": (f"row-block sharded A over {world} GPUs, "
                                       + ("peer-memory push of Q rows (CUDA IPC) + barrier" if p2p
                                          else "NCCL all-gather of Q")),
                       "l2": f"inputs larger than L2: A = {8.0 * cfg.n * cfg.n / 1e9:.2f} GB in total"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": (achieved / hbm_peak) if achieved else None, "traffic": None,
                         "kernel": "A.D on rank 0's rows", "ad_ms_per_launch": ad_ms,
                         "ad_launches_timed": mv_n, "peak_source": peak_src},
            "e2e": {"value": e2e_iters / float(e2e_s.item()), "unit": "iterations/s",
                    "h2d_bytes_per_step": (cfg.n + cfg.n * cfg.p) * 8,
                    "d2h_bytes_per_step": (cfg.n * cfg.p + iters // max(args.steps, 1) * cfg.p) * 8},
            "gpu_launches": launches,
            "clocks": sampler.summary() if hasattr(sampler, "summary") else None,
        }
        print(json.dumps(line))
    eng.close()
    dist.destroy_process_group()
    return 0
