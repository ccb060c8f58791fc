"""Golden hashes of the reference's own problem generator (make_problem<double>).

Run HERE (the container with /root/reference): it calls the UNMODIFIED
reference headers compiled into oracle/_ref/libccgref.so (`make -C oracle ref`)
and writes tests/golden/refgen_hashes.json: for each (n, p, cond, seed) the
SHA-256 of A (row-major float64 bytes), of the spectrum, of b and of X0
(column-major), plus a few sentinel values.  The GPU tests regenerate A on the
device (coopcg_gpu_gen_A(..., COOPCG_MATRIX_RANDOM_SPD, ...)) and compare the
hashes, so sizes the small .npz fixtures cannot hold are still pinned to the
reference bit for bit.

    python tests/golden/make_refgen_hashes.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

CASES = [  # (n, p, cond, seed)
    (33, 2, 1.0, 3),        # cond 1: every spectrum draw equal -> front/back clamp
    (200, 3, 10.0, 11),
    (777, 4, 1e4, 5),       # n not a multiple of the 32-row ring / 64-entry tiles
    (1024, 8, 1e3, 7),
    (2048, 4, 1e2, 1204),
    (4800, 4, 1e2, 3),      # 150 column blocks > 148 SMs: the two-CTAs-per-SM P kernel (~5 min here)
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main() -> None:
    out = []
    for n, p, cond, seed in CASES:
        t0 = time.time()
        A, lam = po.ref_random_spd(n, cond, seed)
        A2, b, X0 = po.ref_make_problem(n, p, cond, seed)
        assert np.array_equal(A, A2)
        out.append({
            "n": n, "p": p, "cond": cond, "seed": seed,
            "A_sha256": sha(A), "spectrum_sha256": sha(lam), "b_sha256": sha(b),
            "X0_colmajor_sha256": sha(np.asarray(X0).T),
            "A00": float(A[0, 0]), "A01": float(A[0, 1]), "A_last": float(A[-1, -1]),
            "lambda_min": float(lam.min()), "lambda_max": float(lam.max()),
        })
        print(f"n={n} cond={cond} seed={seed}: {time.time() - t0:.1f} s", flush=True)
    with open(os.path.join(HERE, "refgen_hashes.json"), "w") as f:
        json.dump({"generator": "reference make_problem<double> via oracle/_ref/libccgref.so",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
