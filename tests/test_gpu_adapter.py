"""The C++ drop-in, run: oracle/_ref/adapter_test (tests/cpp/adapter_test.cpp)
drives the unmodified reference's dysparse::SparsifierState and
dyg::DysparseGpuSparsifierState (include/dyg_dysparse.hpp over libdyg.so)
side by side on the reference's own types -- C2, mixed batches, a failing
batch, usage errors, immediate mode -- and exits non-zero on any difference
in reports, per-event decisions, rows, counters or errors."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "adapter_test")


def test_cpp_adapter_side_by_side():
    assert os.path.exists(BIN), "adapter_test not built (python -c 'import __graft_entry__ as g; g.build()')"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, DYSPARSE_THREADS=str(os.cpu_count() or 1)))
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adapter_test ok" in r.stdout
