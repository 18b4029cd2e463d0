"""Python mirror of the reference's public interface for the update path.

Same names, argument meanings and error behaviour as the reference C++ API
(/root/reference/proj/src): DynamicGraph (graph.hpp:23-68), WalkConfig
(walk.hpp:13-18), SparsifierOptions / SparsifierState / BatchReport
(sparsifier.hpp:25-112), UpdateStream and its file format (stream.hpp),
MatrixMarket I/O (matrix_market.hpp) and run_batch (walk.hpp:86-92).
SparsifierState keeps G and H on the GPU (libdyg.so, include/dyg.h); the
host side never recomputes anything, and there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from ._lib import EVENT_DTYPE, QUERY_DTYPE, REPORT_DTYPE, RESULT_DTYPE, STATS_DTYPE, ptr


class ErrorKind(enum.IntEnum):
    """error.hpp:9 (Device has no reference analogue: CUDA failures)."""
    Usage = 1
    Data = 2
    Numeric = 3
    Device = 4


class Error(RuntimeError):
    """dysparse::Error (error.hpp:11-20)."""

    def __init__(self, kind: int, message: str):
        super().__init__(message)
        self.kind = ErrorKind(kind)


def _check(status: int) -> None:
    if status != 0:
        raise Error(status, _lib.lib().dyg_last_error().decode())


def _hcheck(status: int) -> None:
    if status != 0:
        raise Error(status, _lib.lib().dygh_last_error().decode())


class InsertionDecision(enum.IntEnum):
    Kept = 0
    Pruned = 1


@dataclass
class DeletionOutcome:
    class Kind(enum.IntEnum):
        GraphOnly = 0
        PathRecovered = 1
        LocalFallback = 2

    kind: "DeletionOutcome.Kind" = Kind.GraphOnly
    edges_added: int = 0


@dataclass
class WalkConfig:
    distortion_threshold: float = 10.0  # K
    step_cap: int = 100                 # T
    walker_count: int = 16              # s
    global_seed: int = 0


@dataclass
class SparsifierOptions:
    walk: WalkConfig = field(default_factory=WalkConfig)
    batched: bool = False
    freeze_sparsifier: bool = False


@dataclass
class StreamGenOptions:
    insert_fraction: float = 0.0
    delete_fraction: float = 0.0
    batches: int = 1
    seed: int = 0
    locality: int = 0


@dataclass
class BatchReport:
    batch_index: int = 0
    insertions_seen: int = 0
    insertions_kept: int = 0
    insertions_pruned: int = 0
    deletions_seen: int = 0
    deletions_in_sparsifier: int = 0
    paths_recovered: int = 0
    edges_recovered: int = 0
    fallback_activations: int = 0
    walker_steps: int = 0
    max_event_steps: int = 0
    wall_ms: float = 0.0
    density_graph: float = 0.0
    density_sparsifier: float = 0.0

    @classmethod
    def from_record(cls, r) -> "BatchReport":
        return cls(**{f.name: r[f.name].item() for f in fields(cls)})


@dataclass
class UpdateReport:
    batches: list = field(default_factory=list)
    final_density_graph: float = 0.0
    final_density_sparsifier: float = 0.0


# --------------------------------------------------------------------- graphs
class DynamicGraph:
    """Host adjacency rows with the reference's mutation semantics."""

    def __init__(self, vertex_count: int | None = None, *, _handle=None):
        L = _lib.lib()
        if _handle is None:
            h = C.c_void_p()
            _hcheck(L.dygh_graph_new(vertex_count, C.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib().dygh_graph_free(h)
            self._h = None

    @classmethod
    def from_rows(cls, row_ptr, ids, w) -> "DynamicGraph":
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ids = np.ascontiguousarray(ids, np.uint32)
        w = np.ascontiguousarray(w, np.float64)
        c = _lib.Csr(len(rp) - 1, 0, rp.ctypes.data, ids.ctypes.data if ids.size else 0,
                     w.ctypes.data if w.size else 0)
        h = C.c_void_p()
        _hcheck(_lib.lib().dygh_graph_from_csr(C.byref(c), C.byref(h)))
        return cls(_handle=h)

    def vertex_count(self) -> int:
        return _lib.lib().dygh_graph_n(self._h)

    def edge_count(self) -> int:
        return _lib.lib().dygh_graph_edges(self._h)

    def density(self) -> float:
        return _lib.lib().dygh_graph_density(self._h)

    def insert_edge(self, u: int, v: int, weight: float) -> None:
        _hcheck(_lib.lib().dygh_graph_insert(self._h, u, v, weight))

    def delete_edge(self, u: int, v: int) -> None:
        _hcheck(_lib.lib().dygh_graph_delete(self._h, u, v))

    def edge_weight(self, u: int, v: int) -> float:
        return _lib.lib().dygh_graph_edge_weight(self._h, u, v)

    def has_edge(self, u: int, v: int) -> bool:
        return self.edge_weight(u, v) != 0.0

    def csr(self) -> _lib.Csr:
        """Row-order view (valid until the next mutation)."""
        c = _lib.Csr()
        _hcheck(_lib.lib().dygh_graph_csr(self._h, C.byref(c)))
        return c

    def rows(self):
        """(row_ptr u64[n+1], ids u32[2m], w f64[2m]) copies, reference row order."""
        c = self.csr()
        n = c.n
        rp = np.ctypeslib.as_array(C.cast(c.row_ptr, C.POINTER(C.c_uint64)), (n + 1,)).copy()
        m2 = int(rp[-1])
        if m2 == 0:
            return rp, np.zeros(0, np.uint32), np.zeros(0, np.float64)
        ids = np.ctypeslib.as_array(C.cast(c.ids, C.POINTER(C.c_uint32)), (m2,)).copy()
        w = np.ctypeslib.as_array(C.cast(c.w, C.POINTER(C.c_double)), (m2,)).copy()
        return rp, ids, w

    def neighbors(self, u: int):
        rp, ids, w = self.rows()
        return list(zip(ids[rp[u]:rp[u + 1]].tolist(), w[rp[u]:rp[u + 1]].tolist()))

    def degree(self, u: int) -> int:
        rp, _, _ = self.rows()
        return int(rp[u + 1] - rp[u])


def _graph_from(fn, *args) -> DynamicGraph:
    h = C.c_void_p()
    _hcheck(fn(*args, C.byref(h)))
    return DynamicGraph(_handle=h)


def make_mesh(rows, cols, seed, w_min=0.5, w_max=2.0) -> DynamicGraph:
    return _graph_from(_lib.lib().dygh_make_mesh, rows, cols, seed, w_min, w_max)


def make_grid4(rows, cols, seed, w_min=0.5, w_max=2.0) -> DynamicGraph:
    return _graph_from(_lib.lib().dygh_make_grid4, rows, cols, seed, w_min, w_max)


def make_random_connected(n, extra_edges, seed, w_min=0.1, w_max=10.0, with_pendant=False):
    return _graph_from(_lib.lib().dygh_make_random_connected, n, extra_edges, seed, w_min, w_max,
                       int(with_pendant))


def build_initial_sparsifier(g: DynamicGraph, target_density: float, seed: int) -> DynamicGraph:
    return _graph_from(_lib.lib().dygh_build_initial_sparsifier, g._h, target_density, seed)


def build_initial_sparsifier_gpu(g: DynamicGraph, target_density: float, seed: int,
                                 device: int = 0) -> DynamicGraph:
    """build_initial_sparsifier (sparsifier.cpp:105-159) on the GPU
    (dyg_build_initial_sparsifier), bit-identical to the host builder."""
    c = g.csr()
    n = c.n
    nnz = int(np.ctypeslib.as_array(C.cast(c.row_ptr, C.POINTER(C.c_uint64)), (n + 1,))[n]) \
        if n else 0
    rp = np.zeros(n + 1, np.uint64)
    ids = np.zeros(max(nnz, 1), np.uint32)
    w = np.zeros(max(nnz, 1), np.float64)
    _check(_lib.lib().dyg_build_initial_sparsifier(C.byref(c), float(target_density), int(seed),
                                                   int(device), ptr(rp), ptr(ids), ptr(w)))
    m = int(rp[n])
    return DynamicGraph.from_rows(rp, ids[:m], w[:m])


def load_matrix_market(path: str) -> DynamicGraph:
    return _graph_from(_lib.lib().dygh_load_matrix_market, path.encode())


def save_matrix_market(g: DynamicGraph, path: str) -> None:
    _hcheck(_lib.lib().dygh_save_matrix_market(g._h, path.encode()))


# -------------------------------------------------------------------- streams
class UpdateStream:
    """stream.hpp:20-23: events (numpy EVENT_DTYPE records) + batch_count."""

    def __init__(self, events=None, batch_count: int = 0):
        # Events live in page-locked host memory, so replaying a batch DMAs
        # it straight to the device (no staging copy on the host).
        src = np.zeros(0, EVENT_DTYPE) if events is None else np.asarray(events)
        self.events = _lib.pinned_empty(len(src), EVENT_DTYPE)
        if len(src):
            self.events[:] = np.ascontiguousarray(src, EVENT_DTYPE)
        self.batch_count = int(batch_count)

    @classmethod
    def _from_handle(cls, h) -> "UpdateStream":
        L = _lib.lib()
        n = L.dygh_stream_size(h)
        s = cls(None, L.dygh_stream_batches(h))
        s.events = _lib.pinned_empty(n, EVENT_DTYPE)
        if n:
            src = L.dygh_stream_events(h)
            C.memmove(s.events.ctypes.data, src, n * EVENT_DTYPE.itemsize)
        L.dygh_stream_free(h)
        return s

    def batch_offsets(self):
        """Batch b = events[off[b]:off[b+1]] when the events are grouped by
        batch (the generator's and loader's order), else None. Cached."""
        key = (self.events.ctypes.data, len(self.events), self.batch_count)
        if getattr(self, "_off_key", None) != key:
            bi = self.events["batch_index"]
            off = None
            if len(bi) == 0 or (bool(np.all(bi[1:] >= bi[:-1])) and int(bi[-1]) < self.batch_count):
                off = np.searchsorted(bi, np.arange(self.batch_count + 1)).astype(np.uint64)
            self._off, self._off_key = off, key
        return self._off

    def kind_counts(self):
        """(insertions, deletions) per batch, numpy arrays of batch_count.
        Cached like batch_offsets()."""
        key = (self.events.ctypes.data, len(self.events), self.batch_count)
        if getattr(self, "_kc_key", None) != key:
            k = np.asarray(self.events["kind"])
            bi = np.asarray(self.events["batch_index"]).astype(np.int64)
            nb = self.batch_count
            ins = np.bincount(bi[k == 0], minlength=nb)[:nb]
            self._kc = (ins, np.bincount(bi, minlength=nb)[:nb] - ins)
            self._kc_key = key
        return self._kc

    def batch(self, b: int):
        """(events, positions) of batch b, in stream order. A batch stored
        contiguously (the usual case) is returned as a view of the stream's
        page-locked buffer."""
        pos = np.nonzero(self.events["batch_index"] == b)[0].astype(np.uint64)
        if len(pos) and int(pos[-1]) - int(pos[0]) + 1 == len(pos):
            return self.events[int(pos[0]):int(pos[-1]) + 1], pos
        return np.ascontiguousarray(self.events[pos]), pos


def load_update_stream(path: str) -> UpdateStream:
    h = C.c_void_p()
    _hcheck(_lib.lib().dygh_load_stream(path.encode(), C.byref(h)))
    return UpdateStream._from_handle(h)


def save_update_stream(s: UpdateStream, path: str) -> None:
    L = _lib.lib()
    h = C.c_void_p()
    _hcheck(L.dygh_stream_from_events(ptr(s.events), len(s.events), s.batch_count, C.byref(h)))
    try:
        _hcheck(L.dygh_save_stream(h, path.encode()))
    finally:
        L.dygh_stream_free(h)


def generate_update_stream_gpu(g: DynamicGraph, options: StreamGenOptions,
                               device: int = 0) -> UpdateStream:
    """generate_update_stream with the insertion sampling on the device
    (dyg_generate_stream); locality > 0 uses the host generator."""
    if options.locality:
        return generate_update_stream(g, options)
    L = _lib.lib()
    c = g.csr()
    n, nb = C.c_size_t(), C.c_uint32()
    n_ins = int(round(options.insert_fraction * g.vertex_count()))
    cap = n_ins + int(round(options.delete_fraction * g.edge_count())) + 16
    while True:
        out = _lib.pinned_empty(cap, EVENT_DTYPE)
        st = L.dyg_generate_stream(C.byref(c), options.insert_fraction, options.delete_fraction,
                                   options.batches, options.seed, device, ptr(out), cap,
                                   C.byref(n), C.byref(nb))
        if st == 1 and n.value > cap:
            cap = n.value
            continue
        _check(st)
        break
    s = UpdateStream(None, nb.value)
    s.events = out[:n.value]
    return s


def generate_update_stream(g: DynamicGraph, options: StreamGenOptions) -> UpdateStream:
    h = C.c_void_p()
    _hcheck(_lib.lib().dygh_generate_stream(
        g._h, options.insert_fraction, options.delete_fraction, options.batches, options.seed,
        options.locality, C.byref(h)))
    return UpdateStream._from_handle(h)


# ---------------------------------------------------------------------- state
def _options_struct(o: SparsifierOptions) -> _lib.Options:
    w = o.walk
    return _lib.Options(_lib.WalkCfg(w.distortion_threshold, w.step_cap, w.walker_count,
                                     w.global_seed), int(o.batched), int(o.freeze_sparsifier))


class Decision(enum.IntEnum):
    """DYG_DECISION_* (include/dyg.h): InsertionDecision (sparsifier.hpp:36)
    for insertions, 2 + DeletionOutcome::Kind (sparsifier.hpp:38-42) for
    deletions; NONE for events that did not commit."""
    Kept = 0
    Pruned = 1
    GraphOnly = 2
    PathRecovered = 3
    LocalFallback = 4
    NONE = 255


def _dec_ptr(decisions):
    if decisions is None:
        return None
    if not (isinstance(decisions, np.ndarray) and decisions.dtype == np.uint8
            and decisions.flags.c_contiguous and decisions.flags.writeable):
        raise TypeError("decisions must be a writeable contiguous uint8 numpy array")
    return ptr(decisions)


def ipc_open(handle: bytes, device: int) -> int:
    """Map a peer rank's exchange area (its 64-byte CUDA IPC handle)."""
    p = C.c_void_p()
    buf = (C.c_uint8 * 64).from_buffer_copy(handle)
    _check(_lib.lib().dyg_ipc_open(buf, device, C.byref(p)))
    return p.value


def ipc_close(p: int) -> None:
    _check(_lib.lib().dyg_ipc_close(C.c_void_p(p)))


class SparsifierState:
    """sparsifier.hpp:71-112 with G and H device-resident on `device`."""

    def __init__(self, graph: DynamicGraph, sparsifier: DynamicGraph,
                 options: SparsifierOptions, device: int = 0):
        L = _lib.lib()
        self._options = options
        self._s = None
        self._shard_keep = []
        g, h = graph.csr(), sparsifier.csr()
        opt = _options_struct(options)
        s = C.c_void_p()
        _check(L.dyg_session_create(C.byref(g), C.byref(h), C.byref(opt), device, C.byref(s)))
        self._s = s
        self._n = graph.vertex_count()

    def close(self) -> None:
        if self._s:
            _lib.lib().dyg_session_destroy(self._s)
            self._s = None

    def __del__(self):
        self.close()

    def options(self) -> SparsifierOptions:
        return self._options

    @property
    def update_counter(self) -> int:
        return _lib.lib().dyg_update_counter(self._s)

    def last_event_steps(self) -> int:
        return _lib.lib().dyg_last_event_steps(self._s)

    def info(self, which: int):
        n, e, d = C.c_uint32(), C.c_uint64(), C.c_double()
        _check(_lib.lib().dyg_graph_info(self._s, which, C.byref(n), C.byref(e), C.byref(d)))
        return n.value, e.value, d.value

    def rows(self, which: int):
        """Device rows exported in row order: which 0 = G, 1 = H."""
        n, e, _ = self.info(which)
        rp = np.zeros(n + 1, np.uint64)
        ids = np.zeros(max(2 * e, 1), np.uint32)
        w = np.zeros(max(2 * e, 1), np.float64)
        _check(_lib.lib().dyg_export_rows(self._s, which, ptr(rp), ptr(ids), ptr(w), 2 * e))
        return rp, ids[:2 * e], w[:2 * e]

    def graph(self) -> DynamicGraph:
        return DynamicGraph.from_rows(*self.rows(0))

    def sparsifier(self) -> DynamicGraph:
        return DynamicGraph.from_rows(*self.rows(1))

    def apply_insertion(self, u: int, v: int, weight: float) -> InsertionDecision:
        d = C.c_int()
        _check(_lib.lib().dyg_apply_insertion(self._s, u, v, weight, C.byref(d)))
        return InsertionDecision(d.value)

    def apply_deletion(self, u: int, v: int) -> DeletionOutcome:
        k, a = C.c_int(), C.c_uint32()
        _check(_lib.lib().dyg_apply_deletion(self._s, u, v, C.byref(k), C.byref(a)))
        return DeletionOutcome(DeletionOutcome.Kind(k.value), a.value)

    def replay_batch(self, stream: UpdateStream, batch_index: int,
                     decisions: np.ndarray | None = None) -> BatchReport:
        """sparsifier.cpp:541-548. `decisions` (optional uint8 array, one
        entry per event of the batch) receives each event's DYG_DECISION_*
        (Decision) in stream order."""
        rep = np.zeros(1, REPORT_DTYPE)
        ev = stream.events
        if decisions is not None and len(decisions) < len(stream.batch(batch_index)[0]):
            raise ValueError("decisions needs one entry per event of the batch")
        _check(_lib.lib().dyg_replay_batch(self._s, ptr(ev), len(ev), stream.batch_count,
                                           batch_index, ptr(rep), _dec_ptr(decisions)))
        return BatchReport.from_record(rep[0])

    def replay_events(self, events: np.ndarray, positions: np.ndarray | None,
                      batch_index: int, decisions: np.ndarray | None = None) -> BatchReport:
        """One already-extracted batch (events in stream order)."""
        ev = np.ascontiguousarray(events, EVENT_DTYPE)
        pos = None if positions is None else np.ascontiguousarray(positions, np.uint64)
        rep = np.zeros(1, REPORT_DTYPE)
        if decisions is not None and len(decisions) < len(ev):
            raise ValueError("decisions needs one entry per event")
        _check(_lib.lib().dyg_replay_events(self._s, ptr(ev), ptr(pos) if pos is not None else None,
                                            len(ev), batch_index, ptr(rep), _dec_ptr(decisions)))
        return BatchReport.from_record(rep[0])

    def replay(self, stream: UpdateStream, decisions: np.ndarray | None = None) -> UpdateReport:
        """sparsifier.cpp:550-559. One library call: the host stream's upload
        is pipelined with the batches (dyg_replay_stream). `decisions`
        (optional uint8 array, one entry per stream event) receives every
        event's DYG_DECISION_*, indexed by stream position."""
        out = UpdateReport()
        n = stream.batch_count
        if decisions is not None and len(decisions) < len(stream.events):
            raise ValueError("decisions needs one entry per stream event")
        if n:
            off = stream.batch_offsets()
            rep = np.zeros(n, REPORT_DTYPE)
            _check(_lib.lib().dyg_replay_stream(
                self._s, ptr(stream.events), len(stream.events),
                ptr(off) if off is not None else None, n, ptr(rep), _dec_ptr(decisions)))
            out.batches = [BatchReport.from_record(r) for r in rep]
        out.final_density_graph = self.info(0)[2]
        out.final_density_sparsifier = self.info(1)[2]
        return out

    # dyGRASS.incremental() / .decremental()
    def incremental(self, stream: UpdateStream, batch_index: int) -> BatchReport:
        return self.replay_batch(stream, batch_index)

    def decremental(self, stream: UpdateStream, batch_index: int) -> BatchReport:
        return self.replay_batch(stream, batch_index)

    def upload_stream(self, stream: UpdateStream) -> None:
        """Device-resident copy of the stream. A stream grouped by batch
        uploads asynchronously, batch by batch (dyg_stream_upload_batches);
        the stream must then outlive the uploaded replays."""
        off = stream.batch_offsets()
        if off is not None and stream.batch_count:
            self._uploaded = (stream, off)  # the DMA reads them after this returns
            _check(_lib.lib().dyg_stream_upload_batches(self._s, ptr(stream.events),
                                                        len(stream.events), ptr(off),
                                                        stream.batch_count))
            return
        _check(_lib.lib().dyg_stream_upload(self._s, ptr(stream.events), len(stream.events),
                                            stream.batch_count))

    def replay_uploaded(self, batch_index: int) -> BatchReport:
        rep = np.zeros(1, REPORT_DTYPE)
        _check(_lib.lib().dyg_replay_uploaded(self._s, batch_index, ptr(rep)))
        return BatchReport.from_record(rep[0])

    def replay_uploaded_range(self, first: int, count: int,
                              decisions: np.ndarray | None = None) -> list:
        """Batches [first, first+count) of the uploaded stream, enqueued back to
        back with one host sync (the device-side replay()). `decisions`: as in
        replay(), indexed by position in the uploaded stream."""
        rep = np.zeros(max(count, 1), REPORT_DTYPE)
        _check(_lib.lib().dyg_replay_uploaded_range(self._s, first, count, ptr(rep),
                                                    _dec_ptr(decisions)))
        return [BatchReport.from_record(rep[i]) for i in range(count)]

    def snapshot(self) -> None:
        _check(_lib.lib().dyg_session_snapshot(self._s))

    def restore(self) -> None:
        _check(_lib.lib().dyg_session_restore(self._s))

    def save(self, path: str) -> None:
        """Cross-process checkpoint: options, update_counter and both graphs
        in row order (dyg_session_save)."""
        _check(_lib.lib().dyg_session_save(self._s, os.fsencode(path)))

    @classmethod
    def load(cls, path: str, device: int = 0) -> "SparsifierState":
        """Resume a checkpoint written by save(): same rows, same update
        counter, so the rest of a stream replays as it would have."""
        L = _lib.lib()
        s = C.c_void_p()
        _check(L.dyg_session_load(os.fsencode(path), device, C.byref(s)))
        self = cls.__new__(cls)
        self._s = s
        self._shard_keep = []
        opt = _lib.Options()
        _check(L.dyg_session_options(s, C.byref(opt)))
        w = opt.walk
        self._options = SparsifierOptions(
            WalkConfig(w.distortion_threshold, w.step_cap, w.walker_count, w.global_seed),
            bool(opt.batched), bool(opt.freeze_sparsifier))
        self._n = self.info(0)[0]
        return self

    def stats(self) -> dict:
        st = np.zeros(1, STATS_DTYPE)
        _check(_lib.lib().dyg_session_stats(self._s, ptr(st)))
        return {k: st[0][k].item() for k in STATS_DTYPE.names}

    def set_walk_counters(self, on: bool) -> None:
        """Instrumented walk kernels (per-step statistics in stats(); ~6 %
        slower); the results are identical either way."""
        _check(_lib.lib().dyg_session_set_walk_counters(self._s, int(bool(on))))

    def reset_stats(self) -> None:
        _check(_lib.lib().dyg_session_reset_stats(self._s))

    # -- multi-GPU split, driven by parallel.py -------------
    def shard_begin(self, events, positions, batch_index):
        ev = np.ascontiguousarray(events, EVENT_DTYPE)
        pos = np.ascontiguousarray(positions, np.uint64)
        # The library reads them (error messages) until the batch's commit has
        # been reported: shard_commit, or shard_finish for asynchronous commits.
        self._shard_keep.append((ev, pos))
        nr, nm = C.c_uint64(), C.c_uint64()
        _check(_lib.lib().dyg_shard_begin(self._s, ptr(ev), ptr(pos), len(ev), batch_index,
                                          C.byref(nr), C.byref(nm)))
        return nr.value, nm.value

    def shard_begin_uploaded(self, batch_index):
        """shard_begin for a batch of the stream given to upload_stream."""
        nr, nm = C.c_uint64(), C.c_uint64()
        _check(_lib.lib().dyg_shard_begin_uploaded(self._s, int(batch_index), C.byref(nr),
                                                   C.byref(nm)))
        return nr.value, nm.value

    def shard_record_bytes(self, minpath: bool) -> int:
        return _lib.lib().dyg_shard_record_bytes(self._s, int(minpath))

    def shard_walk(self, rank, world, reach_ptr, min_ptr) -> None:
        _check(_lib.lib().dyg_shard_walk(self._s, rank, world, C.c_void_p(reach_ptr),
                                         C.c_void_p(min_ptr)))

    def shard_commit(self, world, reach_ptr, min_ptr) -> BatchReport:
        rep = np.zeros(1, REPORT_DTYPE)
        try:
            _check(_lib.lib().dyg_shard_commit(self._s, world, C.c_void_p(reach_ptr),
                                               C.c_void_p(min_ptr), ptr(rep)))
        finally:
            self._shard_keep.clear()
        return BatchReport.from_record(rep[0])

    def shard_commit_async(self, world, reach_ptr, min_ptr) -> None:
        _check(_lib.lib().dyg_shard_commit_async(self._s, world, C.c_void_p(reach_ptr),
                                                 C.c_void_p(min_ptr)))

    # -- peer-memory exchange (dyg_shard_peer_*) ----------------------------
    def shard_peer_create(self, world: int, max_reach: int, max_minpath: int):
        """(area pointer, bytes, 64-byte IPC handle) of this rank's exchange area."""
        area, nbytes = C.c_void_p(), C.c_size_t()
        handle = (C.c_uint8 * 64)()
        _check(_lib.lib().dyg_shard_peer_create(self._s, world, max_reach, max_minpath,
                                                C.byref(area), C.byref(nbytes), handle))
        return area.value, nbytes.value, bytes(handle)

    def shard_peer_bind(self, rank: int, world: int, areas, timeout_s: float = 30.0) -> None:
        arr = (C.c_void_p * world)(*areas)
        _check(_lib.lib().dyg_shard_peer_bind(self._s, rank, world, arr, timeout_s))

    def shard_peer_range_begin(self, first: int, count: int) -> None:
        _check(_lib.lib().dyg_shard_peer_range_begin(self._s, first, count))

    def shard_peer_range_end(self, count: int):
        rep = np.zeros(max(count, 1), REPORT_DTYPE)
        n = C.c_size_t()
        _check(_lib.lib().dyg_shard_peer_range_end(self._s, ptr(rep), count, C.byref(n)))
        return [BatchReport.from_record(rep[i]) for i in range(n.value)]

    def shard_finish(self, max_reports: int = 256):
        """Reports of the pending asynchronous shard commits, in order."""
        reps = np.zeros(max(int(max_reports), 1), REPORT_DTYPE)
        n = C.c_size_t(0)
        try:
            _check(_lib.lib().dyg_shard_finish(self._s, ptr(reps), int(max_reports),
                                               C.byref(n)))
        finally:
            self._shard_keep.clear()
        return [BatchReport.from_record(reps[i]) for i in range(min(n.value, max_reports))]

    def set_stream(self, cuda_stream_handle: int) -> None:
        _check(_lib.lib().dyg_set_stream(self._s, C.c_void_p(cuda_stream_handle)))


def run_batch(graph: DynamicGraph, queries: np.ndarray, cfg: WalkConfig, device: int = 0):
    """walk.hpp:86-92 on the GPU: (results RESULT_DTYPE[nq], paths u32[nq, T+1])."""
    q = np.ascontiguousarray(queries, QUERY_DTYPE)
    out = np.zeros(len(q), RESULT_DTYPE)
    paths = np.zeros((len(q), cfg.step_cap + 1), np.uint32)
    c = _lib.WalkCfg(cfg.distortion_threshold, cfg.step_cap, cfg.walker_count, cfg.global_seed)
    g = graph.csr()
    _check(_lib.lib().dyg_run_batch(C.byref(g), ptr(q), len(q), C.byref(c), ptr(out), ptr(paths),
                                    device))
    return out, paths


def device_count() -> int:
    return _lib.lib().dyg_device_count()
