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
    n, p, tol_rel, max_iters, every = case[:5]
    algo = case[5] if len(case) > 5 else "ccg"
    A = po.gen_diagdom(n, n) if n % 2 else po.gen_householder(n, 6, 1e3, n)
    b = po.gen_rhs(n, "uniform", n)
    X0 = po.gen_starts(n, p, n)
    if algo == "mccg-dup":  # duplicate start columns: mccg restricts at setup (solvers.hpp:63-76)
        X0[:, 2] = X0[:, 1]
        algo = "mccg"
    opts = SolveOptions(tol=tol_rel * po.seq_norm(b), max_iters=max_iters, recompute_residual_every=every, algo=algo)
    eng = CpuShardEngine(A, b, X0, rank, world)
    ex = RowExchange(n, eng.P, world, rank)
    t = solve_sharded(eng, ex, opts, poll_every=3)
    if rank == 0:
        ref = po.oracle_ccg(A, b, X0, tol=opts.tol, max_iters=max_iters, recompute=every, algo=algo)
        act = ref.extra["active_agents"] if algo == "mccg" else list(range(p))
        ok = (t.status == ref.status and t.iterations == ref.iterations
              and t.converged_agent == ref.converged_agent
              and np.array_equal(t.residual_norms, ref.residual_norms, equal_nan=True)
              and t.active_agents == act
              and np.array_equal(t.final_x, ref.final_x[:, act])
              and np.array_equal(t.final_residual_norms, ref.final_residual_norms, equal_nan=True)
              and np.array_equal(t.initial, ref.initial_residual_norms))
        out.put((ok, t.status, t.iterations, ref.status, ref.iterations, eng.row0, eng.row1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (80, 3, 1e-10, -1, -1),     # even split, converges (Householder family)
    (81, 3, 1e-10, -1, -1),     # uneven split (staged all-gather), diag-dominant
    (60, 4, 0.0, 30, 7),        # fixed iterations with residual recomputations
    (41, 2, 0.0, 12, 1),        # recompute every iteration, uneven split
    (81, 5, 1e-10, -1, -1, "mccg-dup"),  # mccg: restriction at setup, uneven split
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


def _golden_worker(rank, world, port, name, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from conftest import load_golden
    from cpu_shard_engine import CpuShardEngine
    from paper_1204_0069_b200.sharded import RowExchange, solve_sharded
    from paper_1204_0069_b200.solver import SolveOptions
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, z = load_golden(name)
    opts = SolveOptions(tol=float(z["tol"]), max_iters=int(z["max_iters"]),
                        recompute_residual_every=int(z["recompute"]), algo=str(z["algo"]))
    eng = CpuShardEngine(A, z["b"], z["X0"], rank, world)
    t = solve_sharded(eng, RowExchange(A.shape[0], eng.P, world, rank), opts, poll_every=2)
    if rank == 0:
        act = [int(a) for a in z["active_agents"]]
        ok = (t.status == str(z["status"]) and t.iterations == int(z["iterations"])
              and t.converged_agent == int(z["converged_agent"])
              and np.array_equal(t.residual_norms, z["residual_norms"], equal_nan=True)
              and t.active_agents == act
              and np.array_equal(t.final_x, z["final_x"][:, act])
              and np.array_equal(t.final_residual_norms, z["final_residual_norms"], equal_nan=True))
        out.put((ok, t.status, t.iterations, t.active_agents, str(z["status"]), int(z["iterations"]), act))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["mccg_n50_p8", "mccg_exhaustion_cliff", "mccg_duplicate_columns"])
def test_sharded_gloo_world2_mccg_matches_reference(name):
    """mccg_solve sharded over two gloo ranks: every rank restricts its
    replicated blocks identically on each rank drop (solvers.hpp:156-175); the
    trace equals the reference's own (golden fixtures from the compiled
    reference), NaN rows for the dropped agents included."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_golden_worker, args=(r, 2, port, name, out)) for r in range(2)]
    [p.start() for p in procs]
    res = out.get(timeout=240)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    assert res[0], res[1:]
