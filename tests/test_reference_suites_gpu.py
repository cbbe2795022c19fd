"""Drop-in evidence: the reference's OWN unit suites (proj/tests/test_*.cpp)
and acceptance binary, compiled unmodified against the reference headers and
linked with integration/gte_b200_bridge.cpp + libgte_b200.so (integration/
Makefile), run on the GPU. Every hot-path gte:: call in them executes on the
sm_100a kernels; out-of-scope helpers (Matrix, generate_sbm, IO) come from the
reference's own objects."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BUILD = os.path.join(ROOT, "integration", "_build")
UNIT = os.path.join(BUILD, "ref_unit_tests")
ACCEPT = os.path.join(BUILD, "ref_acceptance")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (integration/Makefile needs /root/reference at build time)")


@pytest.mark.parametrize("suite", ["attention", "graph", "partition", "reformation", "parallel", "interleave"])
def test_reference_unit_suite(cuda, suite):
    _need(UNIT)
    r = subprocess.run([UNIT, f"-ts={suite}"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"suite {suite} failed:\n{r.stdout[-3000:]}\n{r.stderr[-6000:]}"
    assert "0 failed" in r.stdout


def test_reference_acceptance(cuda):
    _need(ACCEPT)
    r = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-6000:]
    assert "FAIL" not in out, out[-6000:]
