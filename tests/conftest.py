"""Test configuration.

Markers: `gpu` tests need a CUDA device and call the product through its
C-ABI (libdyg.so); everything else runs on CPU (oracle pinning, host
pipeline, ABI exports, multi-process exchange logic over gloo).
"""
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: larger configs")


@pytest.fixture(scope="session")
def oracle():
    """The CPU checker: the compiled reference when present, else the
    plain-C restatement (both pinned by tests/test_oracle.py)."""
    from oracle import oracle as O
    for which in ("reference", "restate"):
        if O.available(which):
            return O.load(which)
    O.build("restate")
    return O.load("restate")


@pytest.fixture(scope="session")
def restate():
    from oracle import oracle as O
    if not O.available("restate"):
        O.build("restate")
    return O.load("restate")


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle as O
    if not O.available("reference"):
        if os.path.isdir("/root/reference/proj/src"):
            O.build("reference")
        else:
            pytest.skip("reference oracle not built and /root/reference absent")
    return O.load("reference")


@pytest.fixture(scope="session")
def dyg():
    import paper_2505_02741_b200 as D
    return D
