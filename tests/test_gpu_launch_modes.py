"""Launch-path switches do not change results: programmatic dependent launch off
(COOPCG_NO_PDL=1) and A.D launch events on every iteration (COOPCG_MV_EVERY=1)
give the same exact-mode solve, bit for bit.  The switches are read once per
process, so each variant runs in a fresh interpreter."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import json, numpy as np, paper_1204_0069_b200 as m
n, p = 700, 8
with m.GpuContext(n, p) as ctx:
    ctx.gen_A("diagdom", 7)
    b = m.gen_rhs(n, "uniform", 7); X0 = m.gen_starts(n, p, 7)
    ctx.upload(b, X0)
    t = ctx.run(m.SolveOptions(tol=0.0, max_iters=40, recompute_residual_every=9))
print(json.dumps({"x": t.final_x.tobytes().hex(), "norms": t.residual_norms.tobytes().hex(),
                  "it": t.iteration_count()}))
"""


def _solve(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_launch_switches_bitwise():
    base = _solve({})
    assert base["it"] == 40
    for extra in ({"COOPCG_NO_PDL": "1"}, {"COOPCG_MV_EVERY": "1"}, {"COOPCG_MV_EVERY": "0"}):
        assert _solve(extra) == base, extra


FAST_SCRIPT = r"""
import json, numpy as np, paper_1204_0069_b200 as m
out = {}
for n, p in ((700, 8), (900, 16), (600, 32)):
    with m.GpuContext(n, p, arith="fast") as ctx:
        ctx.gen_A("diagdom", n)
        b = m.gen_rhs(n, "uniform", n); X0 = m.gen_starts(n, p, n)
        ctx.upload(b, X0)
        t = ctx.run(m.SolveOptions(tol=0.0, max_iters=30, recompute_residual_every=9))
        t2 = ctx.run(m.SolveOptions(tol=0.0, max_iters=30, recompute_residual_every=9))
    assert np.array_equal(t.final_x, t2.final_x)  # deterministic run to run
    out[f"{n}_{p}"] = {"x": t.final_x.tolist(), "it": t.iteration_count()}
print(json.dumps(out))
"""


def test_fast_fused_iteration_matches_separate_kernels():
    """The fused post-MMA iteration (fast_iter_kernel, one cooperative launch)
    against the separate row / solve / update kernels (COOPCG_NO_FUSE=1): the
    same per-element arithmetic, the Gram reduction in another fixed order, so
    X agrees far inside the fast mode's 1e-8 bar."""
    def run(extra):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", FAST_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        return json.loads(r.stdout.strip().splitlines()[-1])
    import numpy as np
    sep = run({"COOPCG_NO_FUSE": "1"})
    # the default tiling and every rows-per-thread tile shape (COOPCG_FAST_RP;
    # 4 gives fewer tiles than CTAs at these sizes, 1 the one-tile-per-CTA path)
    for extra in ({}, {"COOPCG_FAST_RP": "1"}, {"COOPCG_FAST_RP": "2"}, {"COOPCG_FAST_RP": "4"}):
        fused = run(extra)
        for key in fused:
            assert fused[key]["it"] == sep[key]["it"] == 30
            a, b = np.array(fused[key]["x"]), np.array(sep[key]["x"])
            assert np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)) < 1e-12, (key, extra)


FAST_BITS_SCRIPT = r"""
import json, numpy as np, paper_1204_0069_b200 as m
out = {}
for n, p in ((700, 8), (1300, 4)):
    with m.GpuContext(n, p, arith="fast") as ctx:
        ctx.gen_A("diagdom", n)
        b = m.gen_rhs(n, "uniform", n); X0 = m.gen_starts(n, p, n)
        ctx.upload(b, X0)
        t = ctx.run(m.SolveOptions(tol=0.0, max_iters=25, recompute_residual_every=9))
        res = ctx.timing()["a_l2_resident_bytes"]
    out[f"{n}_{p}"] = {"x": t.final_x.tobytes().hex(), "norms": t.residual_norms.tobytes().hex(),
                       "it": t.iteration_count()}
    out[f"res_{n}_{p}"] = res
print(json.dumps(out))
"""


def test_fast_ad_shapes_and_l2_residency_bitwise():
    """The fast A.D's consumer-warp shape (2 or 4 M-tiles per DMMA warp,
    COOPCG_FAST_MT) and the L2-resident share of A (COOPCG_L2_RES_MB; evict-last
    copies of the first k-tiles of every work unit) change scheduling and cache
    policy only: the fast-mode solve is the same bytes."""
    def run(extra):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, "-c", FAST_BITS_SCRIPT], cwd=ROOT, env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        return json.loads(r.stdout.strip().splitlines()[-1])
    base = run({"COOPCG_FAST_MT": "4", "COOPCG_L2_RES_MB": "0"})
    assert base["res_700_8"] == 0 and base["700_8"]["it"] == 25
    for extra in ({}, {"COOPCG_FAST_MT": "2"}, {"COOPCG_FAST_MT": "2", "COOPCG_L2_RES_MB": "8"},
                  {"COOPCG_FAST_MT": "4", "COOPCG_L2_RES_MB": "4"}):
        got = run(extra)
        if "COOPCG_L2_RES_MB" in extra:
            assert got["res_700_8"] > 0 and got["res_1300_4"] > 0, extra  # the knob took effect
        for key in ("700_8", "1300_4"):
            assert got[key] == base[key], (key, extra)


GUARD_SCRIPT = r"""
import ctypes as C, numpy as np, paper_1204_0069_b200 as m
from paper_1204_0069_b200 import _capi
from cuda.bindings import runtime as rt
n, p = 300, 4
ctx = m.GpuContext(n, p)
ctx.gen_A("diagdom", 3)
ctx.upload(m.gen_rhs(n, "uniform", 3), m.gen_starts(n, p, 3))
t = ctx.run(m.SolveOptions(tol=0.0, max_iters=5))          # clean run: guards intact
ptr, ld = C.c_void_p(), C.c_int()
assert _capi.lib().coopcg_gpu_block(ctx._h, _capi.BLOCK_X, 0, C.byref(ptr), C.byref(ld)) == 0
# one double just past the end of X, as an off-by-one-row kernel would write
err, = rt.cudaMemset(ptr.value + n * ld.value * 8, 0x11, 8)
assert err == rt.cudaError_t.cudaSuccess
try:
    ctx.run(m.SolveOptions(tol=0.0, max_iters=5))
    print("NOT DETECTED")
except m.CudaError as e:
    print("DETECTED", e)
"""


def test_guard_mode_detects_an_overflow():
    """COOPCG_GUARD=1 (the memcheck stand-in: compute-sanitizer is refused on
    the GPU pool) reports a write past the end of a device buffer."""
    env = dict(os.environ, COOPCG_GUARD="1")
    r = subprocess.run([sys.executable, "-c", GUARD_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "DETECTED" in r.stdout and "guard after the buffer" in r.stdout, r.stdout
