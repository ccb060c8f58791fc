"""Quick all-variants smoke on the GPU box: small solves over every A.D and
solve-kernel variant (pipelined P = 4 / 8 A.D, the 64-row P = 8 kernel, the
two-row-per-thread kernel at P = 16 / 32, the fused solve/update passes, a
residual recompute), each checked against the oracle bit for bit, plus one
fast-mode solve:

    python tests/sanitize_smoke.py

Meant to run under compute-sanitizer (tools/sanitize.sh, SANITIZE_SMALL=1);
the GPU pool refuses compute-sanitizer (profiles/r02_sanitizer_closed.txt),
so the same cases run bitwise against the oracle inside the -m gpu suite."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # test infrastructure: the checker only

import paper_1204_0069_b200 as m  # noqa: E402
import pyoracle as po  # noqa: E402

# (n, p): P=4 pipelined (32-row panels), P=8 old kernel (64-row panels) and
# pipelined (128-row panels), P=16 old rpt kernel (32-row panels), P=32 rpt
CASES = [(301, 3), (777, 8), (9601, 8), (700, 16), (300, 24)]


def main():
    small = os.environ.get("SANITIZE_SMALL") == "1"
    for n, p in CASES:
        if small and n > 1000:
            continue
        A = po.gen_diagdom(n, 7)
        b = po.gen_rhs(n, "uniform", 7)
        X0 = po.gen_starts(n, p, 7)
        ot = po.oracle_ccg(A, b, X0, tol=0.0, max_iters=5, recompute=3)
        gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=0.0, max_iters=5, recompute_residual_every=3))
        ok = np.array_equal(gt.residual_norms, ot.residual_norms) and np.array_equal(gt.final_x, ot.final_x)
        print(f"exact n={n} p={p}: {'bitwise ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            return 1
    n, p = 700, 8
    A = po.gen_diagdom(n, 9)
    b = po.gen_rhs(n, "uniform", 9)
    X0 = po.gen_starts(n, p, 9)
    ft = m.ccg_solve(A, b, X0, m.SolveOptions(tol=0.0, max_iters=6, recompute_residual_every=4),
                     m.GpuOptions(arith="fast"))
    print(f"fast n={n} p={p}: {ft.iteration_count()} iterations, status {ft.status}", flush=True)
    # two row shards driven by one process (peer-push Q, event barriers)
    gt = m.ccg_solve(A, b, X0, m.SolveOptions(tol=0.0, max_iters=6, recompute_residual_every=4),
                     m.GpuOptions(devices=[0, 0]))
    ot = po.oracle_ccg(A, b, X0, tol=0.0, max_iters=6, recompute=4)
    ok = np.array_equal(gt.residual_norms, ot.residual_norms) and np.array_equal(gt.final_x, ot.final_x)
    print(f"exact 2 shards n={n} p={p}: {'bitwise ok' if ok else 'MISMATCH'}", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
