"""Time the reference's own generator, random_spd(n, cond, seed), on the device
(coopcg_gpu_gen_A(..., COOPCG_MATRIX_RANDOM_SPD, ...)) against the reference
itself on the host cores (oracle/_ref/libccgref.so: the unmodified headers;
haar_orthogonal is serial, the U Lambda U^T product uses OpenMP).  Prints one
JSON line per n.  The device number is the whole gen_A call: host Gaussians,
upload, MGS, product, symmetrisation into the context's layout.

    python tools/refgen_bench.py [--n 1024 2048 4096 8192] [--cpu-max 2048]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1024, 2048, 4096, 8192])
    ap.add_argument("--cpu-max", type=int, default=2048)
    ap.add_argument("--cond", type=float, default=1e3)
    ap.add_argument("--seed", type=int, default=7)
    a = ap.parse_args()
    import paper_1204_0069_b200 as m
    import pyoracle as po
    for n in a.n:
        with m.GpuContext(n, 2) as ctx:
            ctx.gen_A("random_spd", a.seed + 1, 0, a.cond)  # warm-up (module load, allocations)
            t0 = time.perf_counter()
            ctx.gen_A("random_spd", a.seed, 0, a.cond)
            t_gpu = time.perf_counter() - t0
            A = ctx.get_A() if n <= a.cpu_max else None
        line = {"n": n, "cond": a.cond, "seed": a.seed, "gpu_s": round(t_gpu, 4)}
        if A is not None and po.ref_available():
            t0 = time.perf_counter()
            A_ref, _ = po.ref_random_spd(n, a.cond, a.seed)
            line["cpu_ref_s"] = round(time.perf_counter() - t0, 3)
            line["cpu_threads"] = os.cpu_count()
            line["bitwise_equal"] = bool(np.array_equal(A, A_ref))
            line["speedup"] = round(line["cpu_ref_s"] / t_gpu, 1)
        elif A is not None:
            line["A_sha256"] = hashlib.sha256(A.tobytes()).hexdigest()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
