"""The C++ drop-in (include/coopcg/gpu_ccg.hpp) against the reference's own
ccg_solve through the reference's types: oracle/_ref/dropin_test, built from
the reference headers by `make -C oracle dropin` (where /root/reference
exists) and shipped with the repo snapshot."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


def test_cpp_dropin_bitwise_vs_reference_ccg_solve():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
