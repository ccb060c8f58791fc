"""The multi-GPU orchestrator (paper_1204_0069_b200.sharded) on CPU: two
processes, gloo all-gathers, an oracle-backed shard engine per rank.  The
sharded solve must be bit-identical to the unsharded oracle solve (DESIGN.md
§7: every row's A-chain is local, everything else is replicated)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    import pyoracle as po
    from cpu_shard_engine import CpuShardEngine
    from paper_1204_0069_b200.sharded import RowExchange, solve_sharded
    from paper_1204_0069_b200.solver import SolveOptions
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, p, tol_rel, max_iters, every = case
    A = po.gen_diagdom(n, n) if n % 2 else po.gen_householder(n, 6, 1e3, n)
    b = po.gen_rhs(n, "uniform", n)
    X0 = po.gen_starts(n, p, n)
    opts = SolveOptions(tol=tol_rel * po.seq_norm(b), max_iters=max_iters, recompute_residual_every=every)
    eng = CpuShardEngine(A, b, X0, rank, world)
    ex = RowExchange(n, eng.P, world, rank)
    t = solve_sharded(eng, ex, opts, poll_every=3)
    if rank == 0:
        ref = po.oracle_ccg(A, b, X0, tol=opts.tol, max_iters=max_iters, recompute=every)
        ok = (t.status == ref.status and t.iterations == ref.iterations
              and np.array_equal(t.residual_norms, ref.residual_norms)
              and np.array_equal(t.final_x, ref.final_x)
              and np.array_equal(t.final_residual_norms, ref.final_residual_norms)
              and np.array_equal(t.initial, ref.initial_residual_norms))
        out.put((ok, t.status, t.iterations, ref.status, ref.iterations, eng.row0, eng.row1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (80, 3, 1e-10, -1, -1),     # even split, converges (Householder family)
    (81, 3, 1e-10, -1, -1),     # uneven split (staged all-gather), diag-dominant
    (60, 4, 0.0, 30, 7),        # fixed iterations with residual recomputations
    (41, 2, 0.0, 12, 1),        # recompute every iteration, uneven split
])
def test_sharded_gloo_world2_bitwise(case):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, out)) for r in range(2)]
    [p.start() for p in procs]
    res = out.get(timeout=240)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    ok, status, it, rstatus, rit, r0, r1 = res
    assert ok, (status, it, rstatus, rit)
