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
    fused, sep = run({}), run({"COOPCG_NO_FUSE": "1"})
    for key in fused:
        assert fused[key]["it"] == sep[key]["it"] == 30
        a, b = np.array(fused[key]["x"]), np.array(sep[key]["x"])
        assert np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)) < 1e-12, key
