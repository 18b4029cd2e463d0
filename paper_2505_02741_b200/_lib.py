"""ctypes binding of libdyg.so (include/dyg.h, include/dyg_host.h).

The product path has no fallback: if the CUDA library is missing this module
raises at import-time of any op, and every device call reports a CUDA error
loudly (status 4) when no GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libdyg.so")

# numpy mirrors of the ABI structs (byte-identical layouts).
EVENT_DTYPE = np.dtype(
    [("kind", "<u4"), ("u", "<u4"), ("v", "<u4"), ("batch_index", "<u4"), ("weight", "<f8")]
)
QUERY_DTYPE = np.dtype(
    [("kind", "<u4"), ("p", "<u4"), ("q", "<u4"), ("pad", "<u4"), ("w_pq", "<f8"),
     ("update_id", "<u8")]
)
RESULT_DTYPE = np.dtype(
    [("reached", "<u4"), ("path_len", "<u4"), ("best_estimate", "<f8"),
     ("steps_used", "<u8"), ("resistance", "<f8")]
)
REPORT_FIELDS = (
    "batch_index", "pad", "insertions_seen", "insertions_kept", "insertions_pruned",
    "deletions_seen", "deletions_in_sparsifier", "paths_recovered", "edges_recovered",
    "fallback_activations", "walker_steps", "max_event_steps", "wall_ms", "density_graph",
    "density_sparsifier",
)
REPORT_DTYPE = np.dtype(
    [("batch_index", "<u4"), ("pad", "<u4")]
    + [(f, "<u8") for f in REPORT_FIELDS[2:12]]
    + [(f, "<f8") for f in REPORT_FIELDS[12:]]
)
STATS_FIELDS = (
    ("batches", "u8"), ("kernel_launches", "u8"), ("reach_queries", "u8"),
    ("minpath_queries", "u8"), ("reach_steps", "u8"), ("minpath_steps", "u8"),
    ("reach_row_bytes", "u8"), ("minpath_row_bytes", "u8"), ("reach_ms", "f8"),
    ("minpath_ms", "f8"), ("commit_ms", "f8"), ("total_ms", "f8"), ("commit_rounds", "u8"),
    ("pool_used", "u8"), ("pool_capacity", "u8"), ("h2d_bytes", "u8"), ("d2h_bytes", "u8"),
    ("commit_ms_deletion", "f8"), ("reach_tail_ms", "f8"), ("minpath_tail_ms", "f8"),
    ("commit_rounds_deletion", "u8"), ("flow_ms_promote", "f8"), ("flow_ms_emit", "f8"),
    ("flow_ms_rank", "f8"), ("flow_ms_apply", "f8"), ("flow_ms_reset", "f8"),
    ("graph_launches", "u8"), ("prep_ms", "f8"), ("walk_commit_gap_ms", "f8"),
    ("batch_gap_ms", "f8"), ("minpath_walk_ms", "f8"), ("reach_tail_row_bytes", "u8"),
    ("minpath_tail_row_bytes", "u8"),
)
STATS_DTYPE = np.dtype([(n, "<" + t) for n, t in STATS_FIELDS])


class Csr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("pad", C.c_uint32), ("row_ptr", C.c_void_p),
                ("ids", C.c_void_p), ("w", C.c_void_p)]


class WalkCfg(C.Structure):
    _fields_ = [("distortion_threshold", C.c_double), ("step_cap", C.c_uint32),
                ("walker_count", C.c_uint32), ("global_seed", C.c_uint64)]


class Options(C.Structure):
    _fields_ = [("walk", WalkCfg), ("batched", C.c_int32), ("freeze_sparsifier", C.c_int32)]


class CondOpts(C.Structure):  # dyg_condition_options
    _fields_ = [("method", C.c_int32), ("max_iterations", C.c_uint32), ("tolerance", C.c_double),
                ("dense_cap", C.c_uint32), ("pad", C.c_uint32), ("seed", C.c_uint64)]


class CondEst(C.Structure):  # dyg_condition_estimate
    _fields_ = [("kappa", C.c_double), ("lambda_max", C.c_double), ("lambda_min", C.c_double),
                ("method", C.c_int32), ("iterations_used", C.c_uint32), ("converged", C.c_int32),
                ("pad", C.c_uint32), ("inner_iterations", C.c_uint64)]


class PcgRes(C.Structure):  # dyg_pcg_result
    _fields_ = [("iterations", C.c_uint32), ("converged", C.c_int32),
                ("relative_residual", C.c_double), ("inner_iterations", C.c_uint64),
                ("energy_count", C.c_uint64)]


_LIB = None


def lib() -> C.CDLL:
    """Load libdyg.so (built in-tree by __graft_entry__.build())."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, dbl, i32, sz = (C.c_void_p, C.c_uint32, C.c_uint64, C.c_double, C.c_int,
                                  C.c_size_t)
    pvp = C.POINTER(C.c_void_p)
    sig = {
        "dyg_last_error": (C.c_char_p, []),
        "dyg_version": (C.c_char_p, []),
        "dyg_device_count": (i32, []),
        "dyg_host_alloc": (vp, [sz]),
        "dyg_host_free": (None, [vp]),
        "dyg_session_create": (i32, [C.POINTER(Csr), C.POINTER(Csr), C.POINTER(Options), i32, pvp]),
        "dyg_session_destroy": (None, [vp]),
        "dyg_replay_batch": (i32, [vp, vp, sz, u32, u32, vp, vp]),
        "dyg_replay_events": (i32, [vp, vp, vp, sz, u32, vp, vp]),
        "dyg_stream_upload": (i32, [vp, vp, sz, u32]),
        "dyg_stream_upload_batches": (i32, [vp, vp, sz, vp, u32]),
        "dyg_replay_stream": (i32, [vp, vp, sz, vp, u32, vp, vp]),
        "dyg_replay_uploaded": (i32, [vp, u32, vp]),
        "dyg_replay_uploaded_range": (i32, [vp, u32, u32, vp, vp]),
        "dyg_apply_insertion": (i32, [vp, u32, u32, dbl, C.POINTER(C.c_int)]),
        "dyg_apply_deletion": (i32, [vp, u32, u32, C.POINTER(C.c_int), C.POINTER(C.c_uint32)]),
        "dyg_last_event_steps": (u64, [vp]),
        "dyg_update_counter": (u64, [vp]),
        "dyg_graph_info": (i32, [vp, i32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_double)]),
        "dyg_export_rows": (i32, [vp, i32, vp, vp, vp, u64]),
        "dyg_session_snapshot": (i32, [vp]),
        "dyg_session_restore": (i32, [vp]),
        "dyg_session_save": (i32, [vp, C.c_char_p]),
        "dyg_session_set_walk_counters": (i32, [vp, i32]),
        "dyg_generate_stream": (i32, [C.POINTER(Csr), dbl, dbl, u32, u64, i32, vp, sz, C.POINTER(sz), C.POINTER(C.c_uint32)]),
        "dyg_shard_peer_create": (i32, [vp, i32, u64, u64, pvp, C.POINTER(sz), vp]),
        "dyg_ipc_open": (i32, [vp, i32, pvp]),
        "dyg_ipc_close": (i32, [vp]),
        "dyg_shard_peer_bind": (i32, [vp, i32, i32, vp, dbl]),
        "dyg_shard_peer_range_begin": (i32, [vp, u32, u32]),
        "dyg_shard_peer_range_end": (i32, [vp, vp, sz, C.POINTER(sz)]),
        "dyg_spectral_ordering_stats": (i32, [C.POINTER(C.c_uint64)] * 3),
        "dyg_session_load": (i32, [C.c_char_p, i32, pvp]),
        "dyg_session_options": (i32, [vp, C.POINTER(Options)]),
        "dyg_session_stats": (i32, [vp, vp]),
        "dyg_session_reset_stats": (i32, [vp]),
        "dyg_run_batch": (i32, [C.POINTER(Csr), vp, sz, C.POINTER(WalkCfg), vp, vp, i32]),
        "dyg_build_initial_sparsifier": (i32, [C.POINTER(Csr), dbl, u64, i32, vp, vp, vp]),
        "dyg_set_stream": (i32, [vp, vp]),
        "dyg_condition_options_default": (None, [C.POINTER(CondOpts)]),
        "dyg_condition_number": (i32, [C.POINTER(Csr), C.POINTER(Csr), C.POINTER(CondOpts), i32,
                                       C.POINTER(CondEst)]),
        "dyg_calibrate_budget": (i32, [C.POINTER(Csr), C.POINTER(Csr), dbl, dbl, u64, i32,
                                       C.POINTER(C.c_double)]),
        "dyg_session_condition_number": (i32, [vp, C.POINTER(CondOpts), C.POINTER(CondEst)]),
        "dyg_session_calibrate_budget": (i32, [vp, dbl, dbl, C.POINTER(C.c_double)]),
        "dyg_pcg_solve": (i32, [C.POINTER(Csr), C.POINTER(Csr), u32, vp, dbl, u32, i32, vp,
                                C.POINTER(PcgRes), vp, sz]),
        "dyg_random_rhs": (i32, [u32, u64, vp]),
        "dyg_shard_begin": (i32, [vp, vp, vp, sz, u32, C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64)]),
        "dyg_shard_record_bytes": (sz, [vp, i32]),
        "dyg_shard_begin_uploaded": (i32, [vp, u32, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64)]),
        "dyg_shard_walk": (i32, [vp, i32, i32, vp, vp]),
        "dyg_shard_commit": (i32, [vp, i32, vp, vp, vp]),
        "dyg_shard_commit_async": (i32, [vp, i32, vp, vp]),
        "dyg_shard_finish": (i32, [vp, vp, sz, C.POINTER(C.c_size_t)]),
        "dygh_last_error": (C.c_char_p, []),
        "dygh_graph_new": (i32, [u32, pvp]),
        "dygh_graph_from_csr": (i32, [C.POINTER(Csr), pvp]),
        "dygh_graph_free": (None, [vp]),
        "dygh_graph_n": (u32, [vp]),
        "dygh_graph_edges": (u64, [vp]),
        "dygh_graph_density": (dbl, [vp]),
        "dygh_graph_insert": (i32, [vp, u32, u32, dbl]),
        "dygh_graph_delete": (i32, [vp, u32, u32]),
        "dygh_graph_edge_weight": (dbl, [vp, u32, u32]),
        "dygh_graph_csr": (i32, [vp, C.POINTER(Csr)]),
        "dygh_make_mesh": (i32, [u32, u32, u64, dbl, dbl, pvp]),
        "dygh_make_grid4": (i32, [u32, u32, u64, dbl, dbl, pvp]),
        "dygh_make_random_connected": (i32, [u32, u32, u64, dbl, dbl, i32, pvp]),
        "dygh_build_initial_sparsifier": (i32, [vp, dbl, u64, pvp]),
        "dygh_generate_stream": (i32, [vp, dbl, dbl, u32, u64, u32, pvp]),
        "dygh_load_matrix_market": (i32, [C.c_char_p, pvp]),
        "dygh_save_matrix_market": (i32, [vp, C.c_char_p]),
        "dygh_load_stream": (i32, [C.c_char_p, pvp]),
        "dygh_save_stream": (i32, [vp, C.c_char_p]),
        "dygh_stream_from_events": (i32, [vp, sz, u32, pvp]),
        "dygh_stream_free": (None, [vp]),
        "dygh_stream_size": (sz, [vp]),
        "dygh_stream_batches": (u32, [vp]),
        "dygh_stream_events": (vp, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


class _PinnedBlock:
    """Owner of one dyg_host_alloc block (freed when the last view dies)."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    def __del__(self):
        if self.ptr and _LIB is not None:
            _LIB.dyg_host_free(self.ptr)
            self.ptr = 0


def pinned_empty(n: int, dtype) -> np.ndarray:
    """Uninitialised array in page-locked memory (the C-ABI DMAs event
    batches straight from it); a plain numpy array when no device is
    usable."""
    dtype = np.dtype(dtype)
    nbytes = n * dtype.itemsize
    if nbytes == 0:
        return np.zeros(n, dtype)
    try:
        ptr = lib().dyg_host_alloc(nbytes)
    except (ImportError, OSError):
        ptr = None
    if not ptr:
        return np.zeros(n, dtype)
    owner = _PinnedBlock(ptr, nbytes)
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    buf._dyg_owner = owner  # numpy views keep buf (their base), buf keeps the block
    return np.frombuffer(buf, dtype=dtype, count=n)


# Every symbol include/*.h declares (checked by tests/test_abi.py).
def declared_symbols() -> list[str]:
    import re
    out = []
    for h in ("dyg.h", "dyg_host.h"):
        path = os.path.join(os.path.dirname(PKG), "include", h)
        with open(path) as f:
            text = f.read()
        out += re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(dygh?_\w+)\s*\(", text, re.M)
    return sorted(set(out))


def ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)
