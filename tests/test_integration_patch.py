"""the reference's CLI (tools/coopcg.cpp:139-151) and
bench harness (src/bench.cpp:165-175) gain the GPU backend through
integration/reference_ccg_gpu.patch.  The patch must apply to the
reference's sources and the patched translation units must type-check with
and without COOPCG_WITH_GPU (integration/check_patch.sh; CLI11 and
nlohmann/json are absent from the reference tree, so compile-only stubs stand
in for them).  Needs the reference tree: runs in the build container."""
import os
import subprocess

import pytest

from conftest import ROOT

REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_reference_patch_applies_and_compiles():
    r = subprocess.run(["bash", os.path.join(ROOT, "integration", "check_patch.sh"), REF],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok ") == 4 and "patch applied" in r.stdout
    assert "warning" not in r.stderr, r.stderr
