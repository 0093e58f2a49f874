"""Shared pytest setup: `gpu` marker, import paths, and library availability.

`-m "not gpu"` tests run on a CPU-only box (oracle vs golden vectors, host
logic, ABI symbol checks, gloo multi-rank tests); `-m gpu` tests need an
sm_100 device and call the CUDA path through the C-ABI.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) device; runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def pbdr():
    from paper_2603_14634_b200 import pbdr as m
    m.lib()  # raises loudly when the CUDA library has not been built
    return m


@pytest.fixture(scope="session")
def pyoracle():
    import pyoracle as o
    o.olib()
    return o


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")) as f:
        return json.load(f)["cases"]
