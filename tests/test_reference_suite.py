"""The reference's OWN unit tests for the hot path (proj/tests/test_{geometry,rasterizer,gradients,
losses,map,tracker}.cpp: 84 test cases, ~115k checks), compiled unmodified against the reference
library built here (oracle/Makefile.ref: proj/src + oracle/eigen_lite) and oracle/doctest_lite.
Passing them shows the build the oracle is pinned to behaves as the reference's own suite demands.
CPU only; needs /root/reference (this container)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
MK = os.path.join(os.path.dirname(HERE), "oracle", "Makefile.ref")

pytestmark = pytest.mark.skipif(not os.path.isdir("/root/reference/proj/tests"),
                                reason="the reference tree is only present in the build container")


def test_reference_unit_suite_passes_on_the_reference_build():
    r = subprocess.run(["make", "-s", "-j8", "-f", MK, "check"], capture_output=True, text=True, timeout=1200)
    summary = [line for line in r.stdout.splitlines() if line.startswith("doctest_lite:") or line.startswith("==")]
    print("\n".join(summary))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert sum(1 for line in summary if line.startswith("doctest_lite:") and " 0 failed;" in line) == 6
