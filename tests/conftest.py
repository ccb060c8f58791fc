"""Shared fixtures.  `-m gpu` tests need a B200 and the built CUDA library;
everything else runs on the CPU (oracle, golden fixtures, host logic, ABI
symbol checks, gloo multi-process tests)."""
import glob
import os
import subprocess
import sys

import numpy as np
import pytest

# The reference's OpenMP solver (oracle/_ref) runs one thread per agent, up to
# p = 32 threads on the box's 16 cores: passive waiting keeps oversubscribed
# barriers from spinning.  Must be set before libgomp loads.
os.environ.setdefault("OMP_WAIT_POLICY", "passive")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)


_ensure_oracle()


@pytest.fixture(scope="session")
def po():
    import pyoracle
    return pyoracle


def golden_names():
    return sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    """Inputs (A, b, X0) + expected reference outputs of one fixture."""
    import pyoracle as po
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    kind = str(z["kind"])
    if "A" in z:
        A = z["A"]
    elif kind == "diagdom":
        A = po.gen_diagdom(int(z["n"]), int(z["seed"]))
    elif kind == "householder":
        A = po.gen_householder(int(z["n"]), int(z["m"]), float(z["kappa"]), int(z["seed"]))
    else:
        raise ValueError(kind)
    return A, z
