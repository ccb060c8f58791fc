"""A seeded slice of the randomised parity sweep (tools/fuzz_parity.py) inside the
GPU suite: random shapes at the kernels' panel / tile boundaries, p = 1..32,
three matrix families, tolerance and fixed-iteration runs, every recompute
policy, ccg / mccg, 1-4 row shards, and sessions of several solves on one
resident context -- exact mode bit for bit against the compiled reference
(oracle/_ref), fast mode inside the north star's tolerances.  The long runs
are recorded in profiles/r02_fuzz_parity.txt."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def fz(po):
    if not po.ref_available():
        pytest.skip("oracle/_ref/libccgref.so not built (needs /root/reference at build time)")
    import fuzz_parity
    return fuzz_parity


@pytest.fixture(scope="module")
def m():
    import paper_1204_0069_b200 as mod
    return mod


@pytest.mark.parametrize("seed,multi,cases", [(11, False, 300), (12, True, 100)])
def test_random_cases_match_the_reference(m, po, fz, seed, multi, cases):
    rng = np.random.default_rng(seed)
    ran = 0
    while ran < cases:
        c = fz.draw_case(rng, multi)
        if fz.cost(c) > 3e8:
            continue
        ran += 1
        for arith in ("exact", "fast"):
            why = fz.run_case(m, po, c, arith)
            assert why is None, (arith, c, why)


def test_random_sessions_on_a_resident_context(m, po, fz):
    rng = np.random.default_rng(13)
    for _ in range(100):
        why = fz.run_session(m, po, rng)
        assert why is None, why
    for _ in range(60):
        why = fz.run_session_fast(m, po, rng)
        assert why is None, why
