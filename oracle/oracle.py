"""ctypes front-end for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module. The product package
(paper_2505_02741_b200/) never does: it fails loudly without its CUDA
library instead of falling back here.

Both oracles export the ABI in oracle/oracle_abi.h:

* ``reference`` -- oracle/_ref/libdyg_ref.so: the unmodified reference sources
  (/root/reference/proj/src) compiled by oracle/ref/Makefile.
* ``restate``   -- oracle/_build/libdyg_oracle.so: the plain-C restatement in
  oracle/restate/dyg_oracle.c, pinned against ``reference`` and against the
  golden vectors under tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIBS = {
    "reference": os.path.join(HERE, "_ref", "libdyg_ref.so"),
    "restate": os.path.join(HERE, "_build", "libdyg_oracle.so"),
}

# numpy dtypes mirroring oracle_abi.h (and include/dyg.h: same layouts).
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
REPORT_FIELDS = [
    "batch_index", "pad", "insertions_seen", "insertions_kept", "insertions_pruned",
    "deletions_seen", "deletions_in_sparsifier", "paths_recovered", "edges_recovered",
    "fallback_activations", "walker_steps", "max_event_steps", "wall_ms", "density_graph",
    "density_sparsifier",
]
REPORT_DTYPE = np.dtype(
    [("batch_index", "<u4"), ("pad", "<u4")]
    + [(f, "<u8") for f in REPORT_FIELDS[2:12]]
    + [(f, "<f8") for f in REPORT_FIELDS[12:]]
)
# Integer report fields that must match bit-for-bit (wall_ms excluded).
REPORT_EXACT = REPORT_FIELDS[2:12] + ["density_graph", "density_sparsifier"]


class OracleError(RuntimeError):
    def __init__(self, kind: int, message: str):
        super().__init__(f"[kind {kind}] {message}")
        self.kind = kind
        self.message = message


class _Cfg(C.Structure):
    _fields_ = [("distortion_threshold", C.c_double), ("step_cap", C.c_uint32),
                ("walker_count", C.c_uint32), ("global_seed", C.c_uint64)]


def build(which: str = "all", quiet: bool = True) -> None:
    """Compile the oracle(s). The reference build needs /root/reference."""
    out = subprocess.DEVNULL if quiet else None
    if which in ("all", "restate"):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "restate")], check=True,
                       stdout=out)
    if which in ("all", "reference") and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "ref")], check=True,
                       stdout=out)


def available(which: str) -> bool:
    return os.path.exists(LIBS[which])


_LOADED: dict[str, "Oracle"] = {}


def load(which: str = "restate") -> "Oracle":
    if which not in _LOADED:
        _LOADED[which] = Oracle(which)
    return _LOADED[which]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """One loaded oracle library."""

    def __init__(self, which: str):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle '{which}' not built: {path}")
        self.which = which
        L = self.lib = C.CDLL(path)
        vp, u32, u64, dbl, i32, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double, C.c_int, C.c_size_t
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_last_error_kind": (i32, []),
            "orc_impl_name": (C.c_char_p, []),
            "orc_graph_new": (vp, [u32]),
            "orc_graph_clone": (vp, [vp]),
            "orc_graph_free": (None, [vp]),
            "orc_graph_n": (u32, [vp]),
            "orc_graph_edges": (u64, [vp]),
            "orc_graph_density": (dbl, [vp]),
            "orc_graph_insert": (i32, [vp, u32, u32, dbl]),
            "orc_graph_delete": (i32, [vp, u32, u32]),
            "orc_graph_edge_weight": (dbl, [vp, u32, u32]),
            "orc_graph_export": (None, [vp, vp, vp, vp]),
            "orc_make_mesh": (vp, [u32, u32, u64, dbl, dbl]),
            "orc_make_grid4": (vp, [u32, u32, u64, dbl, dbl]),
            "orc_make_random_connected": (vp, [u32, u32, u64, dbl, dbl, i32]),
            "orc_build_initial_sparsifier": (vp, [vp, dbl, u64]),
            "orc_stream_generate": (vp, [vp, dbl, dbl, u32, u64, u32]),
            "orc_stream_from_events": (vp, [vp, sz, u32]),
            "orc_stream_size": (sz, [vp]),
            "orc_stream_batches": (u32, [vp]),
            "orc_stream_copy": (None, [vp, vp]),
            "orc_stream_free": (None, [vp]),
            "orc_walker_seed": (u64, [u64, u64, u64]),
            "orc_single_walk": (i32, [vp, u32, u32, dbl, dbl, u32, u64, vp, vp, vp, vp, u32, vp]),
            "orc_loop_erase": (sz, [vp, sz, vp]),
            "orc_run_batch": (i32, [vp, vp, sz, C.POINTER(_Cfg), C.c_uint, vp, vp]),
            "orc_state_new": (vp, [vp, vp, C.POINTER(_Cfg), i32, i32]),
            "orc_state_free": (None, [vp]),
            "orc_state_replay_batch": (i32, [vp, vp, u32, vp]),
            "orc_state_graph": (vp, [vp]),
            "orc_state_sparsifier": (vp, [vp]),
            "orc_state_update_counter": (u64, [vp]),
            "orc_load_matrix_market": (vp, [C.c_char_p]),
            "orc_save_matrix_market": (i32, [vp, C.c_char_p]),
            "orc_stream_load": (vp, [C.c_char_p]),
            "orc_stream_save": (i32, [vp, C.c_char_p]),
        }
        if which == "reference":
            sig["orc_state_replay_batch_decisions"] = (i32, [vp, vp, u32, vp, vp])
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args

    # -- errors -----------------------------------------------------------
    def _check(self, status: int) -> None:
        if status != 0:
            raise OracleError(status, self.lib.orc_last_error().decode())

    def _checkp(self, p):
        if not p:
            raise OracleError(self.lib.orc_last_error_kind(), self.lib.orc_last_error().decode())
        return p

    # -- graphs -----------------------------------------------------------
    def graph(self, n: int) -> "Graph":
        return Graph(self, self._checkp(self.lib.orc_graph_new(n)))

    def make_mesh(self, rows, cols, seed, w_min=0.5, w_max=2.0) -> "Graph":
        return Graph(self, self._checkp(self.lib.orc_make_mesh(rows, cols, seed, w_min, w_max)))

    def make_grid4(self, rows, cols, seed, w_min=0.5, w_max=2.0) -> "Graph":
        return Graph(self, self._checkp(self.lib.orc_make_grid4(rows, cols, seed, w_min, w_max)))

    def make_random_connected(self, n, extra, seed, w_min=0.1, w_max=10.0, with_pendant=False):
        return Graph(self, self._checkp(
            self.lib.orc_make_random_connected(n, extra, seed, w_min, w_max, int(with_pendant))))

    def make_path(self, n, weight=1.0) -> "Graph":
        g = self.graph(n)
        for v in range(n - 1):
            g.insert(v, v + 1, weight)
        return g

    def build_initial_sparsifier(self, g: "Graph", density: float, seed: int) -> "Graph":
        return Graph(self, self._checkp(self.lib.orc_build_initial_sparsifier(g.h, density, seed)))

    def load_matrix_market(self, path: str) -> "Graph":
        return Graph(self, self._checkp(self.lib.orc_load_matrix_market(path.encode())))

    # -- streams ----------------------------------------------------------
    def generate_stream(self, g: "Graph", insert_fraction, delete_fraction, batches, seed,
                        locality=0) -> "Stream":
        return Stream(self, self._checkp(self.lib.orc_stream_generate(
            g.h, insert_fraction, delete_fraction, batches, seed, locality)))

    def stream(self, events: np.ndarray, batch_count: int) -> "Stream":
        ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        return Stream(self, self.lib.orc_stream_from_events(_ptr(ev), len(ev), batch_count))

    def load_stream(self, path: str) -> "Stream":
        return Stream(self, self._checkp(self.lib.orc_stream_load(path.encode())))

    # -- walks ------------------------------------------------------------
    def walker_seed(self, global_seed, update_id, walker) -> int:
        return self.lib.orc_walker_seed(global_seed, update_id, walker)

    def single_walk(self, g, p, q, w_pq, budget, cap, rng_seed):
        term, steps, plen = C.c_uint32(), C.c_uint32(), C.c_uint32()
        acc = C.c_double()
        path = np.zeros(cap + 1, np.uint32)
        self._check(self.lib.orc_single_walk(
            g.h, p, q, w_pq, budget, cap, rng_seed, C.byref(term), C.byref(steps),
            C.byref(acc), _ptr(path), cap + 1, C.byref(plen)))
        return dict(terminal=term.value, steps=steps.value, acc=acc.value,
                    path=path[:plen.value].tolist())

    def loop_erase(self, path) -> list[int]:
        a = np.ascontiguousarray(path, np.uint32)
        out = np.zeros(max(len(a), 1), np.uint32)
        n = self.lib.orc_loop_erase(_ptr(a), len(a), _ptr(out))
        return out[:n].tolist()

    def run_batch(self, g, queries: np.ndarray, K, T, s, seed, workers=1):
        q = np.ascontiguousarray(queries, QUERY_DTYPE)
        out = np.zeros(len(q), RESULT_DTYPE)
        paths = np.zeros((len(q), T + 1), np.uint32)
        cfg = _Cfg(K, T, s, seed)
        self._check(self.lib.orc_run_batch(g.h, _ptr(q), len(q), C.byref(cfg), workers,
                                           _ptr(out), _ptr(paths)))
        return out, paths

    # -- state ------------------------------------------------------------
    def state(self, g, h, K=10.0, T=100, s=16, seed=0, batched=True, freeze=False) -> "State":
        cfg = _Cfg(K, T, s, seed)
        return State(self, self._checkp(
            self.lib.orc_state_new(g.h, h.h, C.byref(cfg), int(batched), int(freeze))))


class Graph:
    def __init__(self, orc: Oracle, handle, owned: bool = True):
        self.o, self.h, self.owned = orc, handle, owned

    def __del__(self):
        if self.owned and self.h:
            self.o.lib.orc_graph_free(self.h)
            self.h = None

    @property
    def n(self) -> int:
        return self.o.lib.orc_graph_n(self.h)

    @property
    def edge_count(self) -> int:
        return self.o.lib.orc_graph_edges(self.h)

    def density(self) -> float:
        return self.o.lib.orc_graph_density(self.h)

    def clone(self) -> "Graph":
        return Graph(self.o, self.o.lib.orc_graph_clone(self.h))

    def insert(self, u, v, w) -> None:
        self.o._check(self.o.lib.orc_graph_insert(self.h, u, v, w))

    def delete(self, u, v) -> None:
        self.o._check(self.o.lib.orc_graph_delete(self.h, u, v))

    def edge_weight(self, u, v) -> float:
        return self.o.lib.orc_graph_edge_weight(self.h, u, v)

    def export(self):
        """(row_ptr u64[n+1], ids u32[2m], w f64[2m]) in reference row order."""
        n, m = self.n, self.edge_count
        rp = np.zeros(n + 1, np.uint64)
        ids = np.zeros(2 * m, np.uint32)
        w = np.zeros(2 * m, np.float64)
        self.o.lib.orc_graph_export(self.h, _ptr(rp), _ptr(ids), _ptr(w))
        return rp, ids, w

    def save_matrix_market(self, path: str) -> None:
        self.o._check(self.o.lib.orc_save_matrix_market(self.h, path.encode()))


class Stream:
    def __init__(self, orc: Oracle, handle):
        self.o, self.h = orc, handle

    def __del__(self):
        if self.h:
            self.o.lib.orc_stream_free(self.h)
            self.h = None

    @property
    def batch_count(self) -> int:
        return self.o.lib.orc_stream_batches(self.h)

    def events(self) -> np.ndarray:
        out = np.zeros(self.o.lib.orc_stream_size(self.h), EVENT_DTYPE)
        self.o.lib.orc_stream_copy(self.h, _ptr(out))
        return out

    def save(self, path: str) -> None:
        self.o._check(self.o.lib.orc_stream_save(self.h, path.encode()))


class State:
    def __init__(self, orc: Oracle, handle):
        self.o, self.h = orc, handle

    def __del__(self):
        if self.h:
            self.o.lib.orc_state_free(self.h)
            self.h = None

    def replay_batch(self, stream: Stream, b: int) -> np.void:
        rep = np.zeros(1, REPORT_DTYPE)
        self.o._check(self.o.lib.orc_state_replay_batch(self.h, stream.h, b, _ptr(rep)))
        return rep[0]

    def replay_batch_decisions(self, stream: Stream, b: int):
        """(report, decisions u8[events of batch b]) -- reference build only;
        DYG_DECISION_* codes, 255 for events that did not commit."""
        n = int((stream.events()["batch_index"] == b).sum())
        rep = np.zeros(1, REPORT_DTYPE)
        dec = np.full(max(n, 1), 255, np.uint8)
        try:
            self.o._check(self.o.lib.orc_state_replay_batch_decisions(self.h, stream.h, b,
                                                                     _ptr(rep), _ptr(dec)))
        except OracleError as e:
            e.decisions = dec[:n]  # the events that committed before the error
            raise
        return rep[0], dec[:n]

    def graph(self) -> Graph:
        return Graph(self.o, self.o.lib.orc_state_graph(self.h), owned=False)

    def sparsifier(self) -> Graph:
        return Graph(self.o, self.o.lib.orc_state_sparsifier(self.h), owned=False)

    @property
    def update_counter(self) -> int:
        return self.o.lib.orc_state_update_counter(self.h)


@dataclass
class Config:
    """A SURVEY.md 8(d) benchmark configuration."""
    name: str
    kind: str          # "mesh" | "grid4"
    rows: int
    cols: int
    insert_fraction: float
    delete_fraction: float
    locality: int
    batches: int = 10
    density: float = 0.10
    K: float = 100.0
    T: int = 100
    s: int = 16
    walk_seed: int = 42
    graph_seed: int = 1
    h_seed: int = 1
    stream_seed: int = 7


CONFIGS = {
    "C1": Config("C1", "mesh", 100, 100, 0.25, 0.0, 3),
    "C2": Config("C2", "mesh", 100, 110, 0.25, 0.01, 3),
    "C3": Config("C3", "mesh", 512, 512, 0.25, 0.01, 3),
    "C4": Config("C4", "grid4", 1225, 1225, 0.25, 0.0, 0),
    "C5": Config("C5", "mesh", 2048, 2048, 0.25, 0.01, 0),
}


def build_config(orc: Oracle, cfg: Config):
    """(G, H0, stream) for a config, from the oracle's own generators."""
    if cfg.kind == "mesh":
        g = orc.make_mesh(cfg.rows, cfg.cols, cfg.graph_seed)
    else:
        g = orc.make_grid4(cfg.rows, cfg.cols, cfg.graph_seed)
    h = orc.build_initial_sparsifier(g, cfg.density, cfg.h_seed)
    st = orc.generate_stream(g, cfg.insert_fraction, cfg.delete_fraction, cfg.batches,
                             cfg.stream_seed, cfg.locality)
    return g, h, st
