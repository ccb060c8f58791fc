"""Where the one-shot drop-in call's time goes at cfg 2 (create, set_A with
its first-use pinned staging, solve, destroy)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1204_0069_b200 as m  # noqa: E402
from paper_1204_0069_b200.configs import CONFIGS, make_problem_on_device  # noqa: E402

cfg = CONFIGS[2]
with m.GpuContext(cfg.n, cfg.p) as ctx:
    b, X0, opts = make_problem_on_device(ctx, cfg)
    A = ctx.get_A()
m.ccg_solve(A, b, X0, opts)
for _ in range(2):
    t0 = time.perf_counter()
    m.ccg_solve(A, b, X0, opts)
    t1 = time.perf_counter()
    ctx = m.GpuContext(cfg.n, cfg.p)
    t2 = time.perf_counter()
    ctx.set_A(A)
    t3 = time.perf_counter()
    tr = ctx.solve(b, X0, opts)
    t4 = time.perf_counter()
    ctx.close()
    t5 = time.perf_counter()
    print(f"ccg_solve {1e3*(t1-t0):.1f} ms | create {1e3*(t2-t1):.1f} set_A {1e3*(t3-t2):.1f} "
          f"solve {1e3*(t4-t3):.1f} destroy {1e3*(t5-t4):.1f} ms")
