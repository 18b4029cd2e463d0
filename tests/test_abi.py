"""The C-ABI boundary (include/dyg.h, include/dyg_host.h), CPU only: the
library loads, exports every declared symbol, keeps the struct layouts the
numpy mirrors assume, and maps reference errors to the ErrorKind status
codes before touching a device."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_2505_02741_b200 import _lib

LIB = _lib.LIB_PATH


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 45, declared
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(L, s)
    # nothing internal leaks (visibility=hidden)
    leaked = [s for s in exported if s.startswith("_ZN3dyg")]
    assert not leaked, leaked[:5]


def test_struct_layouts():
    assert _lib.EVENT_DTYPE.itemsize == 24
    assert _lib.QUERY_DTYPE.itemsize == 32
    assert _lib.RESULT_DTYPE.itemsize == 32
    assert _lib.REPORT_DTYPE.itemsize == 8 + 10 * 8 + 3 * 8
    assert C.sizeof(_lib.Csr) == 32
    assert C.sizeof(_lib.WalkCfg) == 24
    assert C.sizeof(_lib.Options) == 32
    assert _lib.STATS_DTYPE.itemsize == 8 * len(_lib.STATS_FIELDS)


def test_header_compiles_as_c_and_cpp(tmp_path):
    inc = os.path.join(os.path.dirname(os.path.dirname(LIB)), "include")
    src = tmp_path / "t.c"
    src.write_text('#include "dyg.h"\n#include "dyg_host.h"\n'
                   "_Static_assert(sizeof(dyg_event) == 24, \"event\");\n"
                   "_Static_assert(sizeof(dyg_batch_report) == 112, \"report\");\n"
                   "int main(void) { return dyg_version() == 0; }\n")
    subprocess.run(["gcc", "-std=c11", "-I", inc, "-c", str(src), "-o", str(tmp_path / "t.o")],
                   check=True)
    cpp = tmp_path / "t.cpp"
    cpp.write_text('#include "dyg_host.hpp"\nint main() { dyg::WalkConfig c; return c.step_cap != 100; }\n')
    subprocess.run(["g++", "-std=c++20", "-I", inc, "-c", str(cpp), "-o", str(tmp_path / "u.o")],
                   check=True)


def test_version_and_device_count():
    L = _lib.lib()
    assert b"sm_100a" in L.dyg_version()
    assert L.dyg_device_count() >= 0


def csr_of(g):
    return g.csr()


def test_session_ctor_validation_before_device(dyg):
    # sparsifier.cpp:183-203 checks run on the host, before any CUDA call.
    L = _lib.lib()
    g = dyg.make_mesh(4, 4, 1)
    h_bad_n = dyg.DynamicGraph(15)
    opt = _lib.Options(_lib.WalkCfg(10.0, 100, 16, 0), 1, 0)
    s = C.c_void_p()
    gc, hc = g.csr(), h_bad_n.csr()
    assert L.dyg_session_create(C.byref(gc), C.byref(hc), C.byref(opt), 0, C.byref(s)) == 1
    assert b"share a vertex set" in L.dyg_last_error()
    h = dyg.DynamicGraph(16)
    h.insert_edge(0, 15, 1.0)
    hc = h.csr()
    assert L.dyg_session_create(C.byref(gc), C.byref(hc), C.byref(opt), 0, C.byref(s)) == 2
    assert L.dyg_last_error() == b"sparsifier edge (0, 15) missing from the graph"
    bad = _lib.Options(_lib.WalkCfg(-1.0, 100, 16, 0), 1, 0)
    hc = dyg.DynamicGraph(16).csr()
    assert L.dyg_session_create(C.byref(gc), C.byref(hc), C.byref(bad), 0, C.byref(s)) == 1
    assert L.dyg_last_error() == b"invalid walk configuration"


def test_run_batch_usage_errors_before_device(dyg):
    from oracle import oracle as O
    g = dyg.DynamicGraph(4)
    g.insert_edge(0, 1, 1.0)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (0, 1, 1, 0, 1.0, 0)
    with pytest.raises(dyg.Error) as e:
        dyg.run_batch(g, q, dyg.WalkConfig())
    assert e.value.kind == dyg.ErrorKind.Usage and "endpoints must differ" in str(e.value)
    q[0] = (0, 9, 1, 0, 1.0, 0)
    with pytest.raises(dyg.Error) as e:
        dyg.run_batch(g, q, dyg.WalkConfig())
    assert str(e.value) == "vertex id 9 out of range (n = 4)"


def test_null_arguments_are_usage_errors():
    L = _lib.lib()
    assert L.dyg_replay_batch(None, None, 0, 0, 0, None, None) == 1
    assert L.dyg_session_snapshot(None) == 1
    assert L.dyg_update_counter(None) == 0
    L.dyg_session_destroy(None)  # no-op
    # round-2 entry points: null / invalid arguments are Usage errors, no device touched
    assert L.dyg_stream_upload_batches(None, None, 0, None, 0) == 1
    assert L.dyg_shard_peer_range_begin(None, 0, 0) == 1
    assert L.dyg_shard_peer_bind(None, 0, 1, None, 1.0) == 1
    assert L.dyg_session_options(None, None) == 1
    assert L.dyg_generate_stream(None, 0.1, 0.0, 1, 1, 0, None, 0, None, None) == 1


def test_dysparse_adapter_compiles_against_reference_headers(tmp_path):
    """include/dyg_dysparse.hpp instantiates the adapter with the reference's
    own types (needs /root/reference for its headers)."""
    ref = "/root/reference/proj"
    if not os.path.isdir(ref):
        pytest.skip("reference headers absent")
    inc = os.path.join(os.path.dirname(os.path.dirname(LIB)), "include")
    repo = os.path.dirname(inc)
    subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-I", inc,
                    "-I", os.path.join(repo, "oracle", "ref"),
                    "-I", os.path.join(repo, "oracle", "ref", "fake_eigen"),
                    "-I", os.path.join(ref, "src"), "-I", os.path.join(ref, "tests"),
                    os.path.join(repo, "tests", "cpp", "adapter_test.cpp")], check=True)


def test_checkpoint_file_errors_before_device(dyg, tmp_path):
    """dyg_session_load reads and checks the whole file before touching a
    device: missing, foreign, truncated and corrupted files are Data errors."""
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState.load(str(tmp_path / "missing.ckpt"))
    assert e.value.kind == dyg.ErrorKind.Data and "cannot open checkpoint" in str(e.value)
    foreign = tmp_path / "foreign.ckpt"
    foreign.write_bytes(b"NOTACKPT" + bytes(64))
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState.load(str(foreign))
    assert e.value.kind == dyg.ErrorKind.Data and "not a checkpoint file" in str(e.value)
    trunc = tmp_path / "trunc.ckpt"
    trunc.write_bytes(b"DYGCKPT1" + bytes(20))
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState.load(str(trunc))
    assert e.value.kind == dyg.ErrorKind.Data and "truncated checkpoint" in str(e.value)
    L = _lib.lib()
    assert L.dyg_session_save(None, b"x") == 1
