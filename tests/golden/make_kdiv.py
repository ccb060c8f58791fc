"""Measure k_div for the BASELINE configs.

TEST-FIXTURE GENERATOR; runs in the build container (it needs the reference
tree to compile oracle/_ref).  Writes tests/golden/kdiv.json.

k_div is the first iteration k at which the reference's own residual-norm
history, computed by two builds of the UNMODIFIED reference headers that
differ only in floating-point contraction (oracle/_ref/libccgref.so with
-ffp-contract=off, the reference's own flag, CMakeLists.txt:25, vs
oracle/_ref/libccgref_fma.so with -march=native -ffp-contract=fast), differs
by more than 1e-8 relative in any agent -- or at which the history reaches the
round-off floor (minres / ||b|| < 1e-12), whichever comes first.  Past k_div
no reordered arithmetic (the GPU fast mode included) can be held to the
north star's 1e-8 history bar, because finite-precision CG is chaotic there
(SURVEY.md §0.6); the fast-mode full-size tests
(tests/test_gpu_full_configs.py) check the history for k < k_div and the
iterates and final residuals everywhere.

    make -C oracle ref ref-fma && python tests/golden/make_kdiv.py [cfg ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import pyoracle as po  # noqa: E402

# The BASELINE configs (paper_1204_0069_b200/configs.py, restated so this
# script needs nothing from the product): n, p, matrix, m, kappa, rel_tol, fixed_iters, seed
CFGS = {
    0: (1000, 3, "diagdom", 0, 1.0, 1e-10, -1, 12040),
    1: (4096, 4, "householder", 8, 1e4, 1e-10, -1, 12041),
    2: (16384, 8, "diagdom", 0, 1.0, 0.0, 200, 12042),
}
FMA_SO = os.path.join(ROOT, "oracle", "_ref", "libccgref_fma.so")


def inputs(n, p, matrix, m, kappa, seed, out):
    if matrix == "diagdom":
        po.gen_diagdom_rows(n, seed, 0, n, out=out)
        b = po.gen_rhs(n, "uniform", seed)
    else:
        po.gen_householder_into(n, m, kappa, seed, out)
        b = po.gen_rhs(n, "normal", seed)
    return b, po.gen_starts(n, p, seed)


def kdiv(t1, t2, nb):
    k = min(t1.iterations, t2.iterations)
    for i in range(k):
        rel = np.max(np.abs(t1.residual_norms[i] - t2.residual_norms[i]) / t1.residual_norms[i])
        if rel > 1e-8 or t1.minres[i] / nb < 1e-12:
            return i, "diverged" if rel > 1e-8 else "floor"
    return k, "end"


def main(which):
    path = os.path.join(HERE, "kdiv.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for c in which:
        n, p, matrix, m, kappa, rel_tol, fixed, seed = CFGS[c]
        t0 = time.time()
        traces = []
        for lib in (po.REF_SO, FMA_SO):
            with po.RefMatrix(n, lib) as R:
                b, X0 = inputs(n, p, matrix, m, kappa, seed, R.A)
                nb = po.seq_norm(b)
                tol = rel_tol * nb if fixed < 0 else 0.0
                traces.append(R.solve(b, X0, tol=tol, max_iters=fixed, algo="parallel"))
        t1, t2 = traces
        k, why = kdiv(t1, t2, nb)
        out[f"cfg{c}"] = {"n": n, "p": p, "k_div": k, "reason": why,
                          "iterations_nofma": t1.iterations, "iterations_fma": t2.iterations,
                          "status_nofma": t1.status, "status_fma": t2.status,
                          "x_rel_diff": float(np.max(np.linalg.norm(t1.final_x - t2.final_x, axis=0)
                                                     / np.linalg.norm(t1.final_x, axis=0)))}
        print(f"cfg{c}: {out[f'cfg{c}']}  ({time.time() - t0:.0f} s)", flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or sorted(CFGS))
