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
