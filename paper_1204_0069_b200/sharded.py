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
    engine.collective_stream() -> context manager ordering collectives with
                                  the engine's stream
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

PH_SETUP_LOCAL, PH_SETUP_REST, PH_ITER_LOCAL, PH_ITER_MID, PH_ITER_REST, PH_FINAL_LOCAL, PH_FINAL_REST = range(7)
BLOCK_X, BLOCK_R, BLOCK_D, BLOCK_Q, BLOCK_S = range(5)


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


def solve_sharded(engine, exchange: RowExchange, opts: SolveOptions, poll_every: int = 8):
    """Drive one sharded solve (the phase protocol of include/coopcg_gpu.h)."""
    engine.begin(opts)
    engine.phase(PH_SETUP_LOCAL, 0)
    with engine.collective_stream():
        exchange.allgather(engine.block(BLOCK_R, 0))
    engine.phase(PH_SETUP_REST, 0)
    stop, _ = engine.state()
    k = 0
    while not stop and k < engine.max_iters:
        engine.phase(PH_ITER_LOCAL, k)
        with engine.collective_stream():
            exchange.allgather(engine.block(BLOCK_Q, k))
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

    def block(self, which: int, k: int):
        ptr = C.c_void_p()
        ld = C.c_int()
        _check(self.ctx._h, _capi.lib().coopcg_gpu_block(self.ctx._h, which, k, C.byref(ptr), C.byref(ld)))
        key = ptr.value
        if key not in self._views:
            self._views[key] = self._torch.as_tensor(_CudaArray(ptr.value, (self.n, self.P), self.device),
                                                     device=f"cuda:{self.device}")
        return self._views[key]

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


def bench_main(args, cfg, metric: str) -> int:
    """bench.py under torchrun: row-sharded solve of `cfg` on WORLD_SIZE GPUs."""
    import torch
    import torch.distributed as dist
    from .configs import host_inputs, solve_options
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if cfg.matrix != "diagdom":
        if rank == 0:
            print(json.dumps({"metric": metric, "unavailable": "sharded Householder generation is not "
                              "implemented this round (diag-dominant configs shard)"}))
        dist.destroy_process_group()
        return 0
    eng = GpuShardEngine(cfg.n, cfg.p, rank, world, local, arith=args.arith)
    eng.ctx.gen_A(cfg.matrix, cfg.seed, cfg.reflectors, cfg.kappa)
    b, X0 = host_inputs(cfg)
    opts = solve_options(cfg, b)
    eng.ctx.upload(b, X0)
    ex = RowExchange(cfg.n, eng.P, world, rank)
    for _ in range(args.warmup):
        solve_sharded(eng, ex, opts)
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    iters = 0
    e0.record(eng._stream)
    for _ in range(args.steps):
        t = solve_sharded(eng, ex, opts)
        iters += t.iteration_count()
    e1.record(eng._stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        secs = float(ms.item()) * 1e-3
        print(json.dumps({
            "metric": metric, "value": iters / secs, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64 generators, DESIGN.md §3)",
            "config": {"workload": cfg.name, "n": cfg.n, "p": cfg.p, "arith": args.arith,
                       "parallelism": f"row-block sharded A over {world} GPUs, NCCL all-gather of Q"},
        }))
    eng.close()
    dist.destroy_process_group()
    return 0
