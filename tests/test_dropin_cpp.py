"""Runs the C++ drop-in API driver (tests/cpp/test_dropin.cpp, built by
__graft_entry__.build()) on the GPU: pbdr::Scene / SolverConfig / step() /
Solver used the way the reference's solver tests would use them."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_dropin")


def test_dropin_driver_built():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_dropin_driver_passes():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all passed" in r.stdout
