"""Peer-memory Q exchange (coopcg_gpu_ipc_handles / coopcg_gpu_set_peers) with
two or three ranks (processes) on one GPU.  Each rank's A.D (exact) or row pass
(fast) stores its rows of Q into every rank's Q through CUDA IPC mappings; the Q
exchange is then only a barrier (stream sync + gloo barrier: no kernel ever
waits on another, the two processes time-share the GPU).  R and S (setup,
recompute, final) travel by a host-staged gloo all-gather.  Exact mode must be
bit-identical to the oracle; fast mode identical on both ranks and within the
fast-mode tolerance of the single-context solve."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, arith, opts_t, inputs_path, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1204_0069_b200 as m
    from paper_1204_0069_b200.sharded import GpuShardEngine, PeerQExchange, solve_sharded

    class HostStagedPeerExchange(PeerQExchange):
        def allgather(self, block):  # R / S: through host memory (gloo has no CUDA all-gather)
            torch.cuda.current_stream().synchronize()
            parts = [None] * self.world
            dist.all_gather_object(parts, (self.r0, block[self.r0:self.r1].cpu().numpy()))
            for r0, rows in parts:
                if r0 != self.r0:
                    block[r0:r0 + rows.shape[0]].copy_(torch.from_numpy(rows))
            torch.cuda.current_stream().synchronize()

    z = np.load(inputs_path)
    A, b, X0 = z["A"], z["b"], z["X0"]
    n, p = A.shape[0], X0.shape[1]
    eng = GpuShardEngine(n, p, rank, world, 0, arith)
    eng.ctx.set_A(A[eng.row0:eng.row1])
    eng.ctx.upload(b, X0)
    eng.enable_peers()
    ex = HostStagedPeerExchange(n, eng.P, world, rank, None, 0)
    tol, max_iters, every = opts_t
    tr = solve_sharded(eng, ex, m.SolveOptions(tol=tol, max_iters=max_iters, recompute_residual_every=every),
                       poll_every=4)
    np.savez(out_path % rank, norms=tr.residual_norms, x=tr.final_x, fres=tr.final_residual_norms,
             it=tr.iteration_count(), status=str(tr.status))
    eng.close()
    dist.destroy_process_group()


def _run(tmp_path, arith, A, b, X0, opts_t, world=2):
    import torch.multiprocessing as mp
    inputs = str(tmp_path / "inputs.npz")
    np.savez(inputs, A=A, b=b, X0=X0)
    out = str(tmp_path / "rank%d.npz")
    mp.start_processes(_worker, args=(world, _free_port(), arith, opts_t, inputs, out), nprocs=world, join=True,
                       start_method="spawn")
    return [np.load(out % r) for r in range(world)]


@pytest.mark.parametrize("n,p,world", [(301, 4, 2), (517, 8, 3)])  # uneven row blocks
def test_peer_q_exchange_exact_bitwise(po, tmp_path, n, p, world):
    A = po.gen_diagdom(n, 41)
    b = po.gen_rhs(n, "uniform", 41)
    X0 = po.gen_starts(n, p, 41)
    opts_t = (0.0, 30, 7)  # 30 iterations, recompute every 7 (R all-gathers between)
    res = _run(tmp_path, "exact", A, b, X0, opts_t, world)
    ref = po.oracle_ccg(A, b, X0, tol=0.0, max_iters=30, recompute=7)
    for r in res:
        assert str(r["status"]) == ref.status and int(r["it"]) == ref.iterations
        assert np.array_equal(r["norms"], ref.residual_norms)
        assert np.array_equal(r["x"], ref.final_x)
        assert np.array_equal(r["fres"], ref.final_residual_norms)


def test_peer_q_exchange_fast(po, tmp_path):
    import paper_1204_0069_b200 as m
    n, p = 700, 8
    A = po.gen_diagdom(n, 43)
    b = po.gen_rhs(n, "uniform", 43)
    X0 = po.gen_starts(n, p, 43)
    opts_t = (0.0, 12, 5)
    res = _run(tmp_path, "fast", A, b, X0, opts_t)
    assert np.array_equal(res[0]["x"], res[1]["x"])  # replicated state on both ranks
    assert np.array_equal(res[0]["norms"], res[1]["norms"])
    single = m.ccg_solve(A, b, X0, m.SolveOptions(tol=0.0, max_iters=12, recompute_residual_every=5),
                         m.GpuOptions(arith="fast"))
    assert int(res[0]["it"]) == single.iteration_count()
    rel = np.linalg.norm(res[0]["x"] - single.final_x) / np.linalg.norm(single.final_x)
    assert rel < 1e-10
