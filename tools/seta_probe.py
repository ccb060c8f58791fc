import time, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_1204_0069_b200 as m
n, p = 16384, 8
A = np.random.default_rng(1).uniform(-1, 1, (n, n))
with m.GpuContext(n, p) as ctx:
    ctx.set_A(A)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); ctx.set_A(A); ts.append(time.perf_counter() - t0)
print(os.environ.get("COOPCG_PIN_MB", "32"), os.environ.get("COOPCG_COPY_THREADS", "8"), f"set_A {min(ts)*1e3:.1f} ms = {A.nbytes/min(ts)/1e9:.1f} GB/s")
t0 = time.perf_counter()
with m.GpuContext(n, p) as ctx: pass
print(f"create+destroy {1e3*(time.perf_counter()-t0):.1f} ms")
