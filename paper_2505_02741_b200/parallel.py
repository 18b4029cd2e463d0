"""Multi-GPU replay: one process per GPU.

Every rank holds a full replica of G and H (SparsifierState on its own
device). For each batch:

  1. every rank builds the same query lists on its replica
     (dyg_shard_begin: validate, walk shadow, query build);
  2. rank r walks the contiguous query range
     [floor(nq*r/P), floor(nq*(r+1)/P)) and packs one fixed-size record per
     query slot (dyg_shard_walk; reach: 16 B {reached, steps}; min-path:
     24 B header + (T+1) path vertices);
  3. the records are exchanged -- the batch's single real exchange step;
  4. every rank applies the identical deterministic commit
     (dyg_shard_commit), so the replicas stay bit-identical.

Two transports for step 3:
  * "peer" (default for uploaded ranges): each rank's records stay in its
    own device exchange area; the ranks map each other's areas once (CUDA
    IPC, handles swapped over torch.distributed) and every rank's kernels
    read the peers' records over NVLink after a per-batch epoch handshake in
    device memory (dyg_shard_peer_*). A whole range of batches is then one
    captured graph per rank with no host step and no collective call.
  * "collective": an all-gather per batch through torch.distributed (NCCL
    on NVLink; gloo stages through host memory), between the library's
    walk and commit calls.

torch.distributed is plumbing only (process group, handle exchange, the
collective transport); the walk, exchange and commit run in libdyg.so.
"""
from __future__ import annotations

import numpy as np


def shard_range(nq: int, rank: int, world: int) -> tuple[int, int]:
    """Query range of `rank` (same formula as dyg_shard_walk)."""
    return nq * rank // world, nq * (rank + 1) // world


def slots_per_rank(nq: int, world: int) -> int:
    return (nq + world - 1) // world


def owner_of(q: int, nq: int, world: int) -> tuple[int, int]:
    """(rank, index within the rank's slots) of query q."""
    r = min(world - 1, q * world // max(nq, 1))
    while r + 1 < world and nq * (r + 1) // world <= q:
        r += 1
    while r > 0 and nq * r // world > q:
        r -= 1
    return r, q - nq * r // world


def allgather_records(local, world: int, group=None):
    """Rank-major all-gather of equal-size record buffers (uint8 tensors)."""
    import torch
    import torch.distributed as dist

    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    if local.numel():
        dist.all_gather_into_tensor(out, local, group=group)
    return out


def unpack_records(gathered: np.ndarray, nq: int, world: int, rec_bytes: int) -> np.ndarray:
    """Host mirror of k_unpack_*: rank-major slots -> query order (tests)."""
    slots = slots_per_rank(nq, world)
    g = gathered.reshape(world * slots, rec_bytes) if nq else gathered.reshape(0, rec_bytes)
    out = np.zeros((nq, rec_bytes), np.uint8)
    for q in range(nq):
        r, i = owner_of(q, nq, world)
        out[q] = g[r * slots + i]
    return out


class ShardedReplay:
    """Drives a SparsifierState replica on this rank's GPU through the
    sharded protocol. `state` must live on torch.cuda.current_device()."""

    def __init__(self, state, rank: int, world: int, group=None, transport: str = "peer",
                 peer_timeout_s: float = 30.0):
        import torch

        self.state, self.rank, self.world, self.group = state, rank, world, group
        self.device = torch.device("cuda", torch.cuda.current_device())
        # Kernels and the collective share one stream (stream-ordered).
        state.set_stream(torch.cuda.current_stream().cuda_stream)
        self.rbytes = state.shard_record_bytes(False)
        self.mbytes = state.shard_record_bytes(True)
        self.bytes_exchanged = 0
        import torch.distributed as dist

        self._nccl = dist.get_backend(group) == "nccl"
        if transport not in ("peer", "collective"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        self.peer_timeout_s = peer_timeout_s
        self._peer_key = None      # (max_reach, max_minpath) the areas were sized for
        self._peer_mapped = []     # IPC mappings of the other ranks' areas
        self._kind_counts = None   # per-batch insertions / deletions of the uploaded stream
        self._bufs = {}  # reused record buffers (grown on demand)

    def _buf(self, key, nbytes):
        import torch

        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            # Zeroed once: the buffers are sized by host-known upper bounds and
            # the pack kernels write only the actual records, so the gather
            # (and gloo's host staging) would otherwise read never-written
            # bytes (compute-sanitizer initcheck).
            b = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=self.device)
            self._bufs[key] = b
        return b[:nbytes]

    def _exchange(self, nr, nm, commit=True):
        sr, sm = slots_per_rank(nr, self.world), slots_per_rank(nm, self.world)
        rloc = self._buf("rloc", sr * self.rbytes)
        mloc = self._buf("mloc", sm * self.mbytes)
        self.state.shard_walk(self.rank, self.world, rloc.data_ptr() if sr else 0,
                              mloc.data_ptr() if sm else 0)
        rall = self._gather("rall", rloc)
        mall = self._gather("mall", mloc)
        self.bytes_exchanged += rall.numel() + mall.numel()
        if not commit:
            # Enqueued only: the record buffers are reused by the next batch in
            # stream order, after this batch's unpack has read them.
            self.state.shard_commit_async(self.world, rall.data_ptr() if sr else 0,
                                          mall.data_ptr() if sm else 0)
            return None
        return self.state.shard_commit(self.world, rall.data_ptr() if sr else 0,
                                       mall.data_ptr() if sm else 0)

    def _gather(self, key, local):
        import torch
        import torch.distributed as dist

        out = self._buf(key, self.world * local.numel())
        if not local.numel():
            return out
        if self._nccl:
            dist.all_gather_into_tensor(out, local, group=self.group)
        else:
            # A host-side backend (gloo: several ranks sharing one GPU in the
            # tests): stage the records through host memory, rank-major as
            # NCCL lays them out.
            host = local.cpu()
            parts = [torch.empty_like(host) for _ in range(self.world)]
            dist.all_gather(parts, host, group=self.group)
            out.copy_(torch.cat(parts).to(out.device))
        return out

    def replay_events(self, events, positions, batch_index: int):
        nr, nm = self.state.shard_begin(events, positions, batch_index)
        return self._exchange(nr, nm)

    def upload(self, stream):
        """dyg_stream_upload of `stream` plus its per-batch kind counts (the
        peer areas are sized from them)."""
        self.state.upload_stream(stream)
        self._kind_counts = stream.kind_counts()

    def replay_uploaded(self, batch_index: int):
        """Batch `batch_index` of the stream given to state.upload_stream."""
        nr, nm = self.state.shard_begin_uploaded(batch_index)
        return self._exchange(nr, nm)

    def _peer_setup(self, max_reach: int, max_minpath: int):
        """Size, publish and map the exchange areas (collective over the
        group: every rank calls it with the same maxima)."""
        import torch
        import torch.distributed as dist

        from .api import ipc_close, ipc_open

        key = (max_reach, max_minpath)
        if self._peer_key is not None and key[0] <= self._peer_key[0] and key[1] <= self._peer_key[1]:
            return
        for p in self._peer_mapped:
            ipc_close(p)
        self._peer_mapped = []
        area, _, handle = self.state.shard_peer_create(self.world, max_reach, max_minpath)
        handles = [None] * self.world
        dist.all_gather_object(handles, handle, group=self.group)
        dev = torch.cuda.current_device()
        areas, err = [], None
        for q, h in enumerate(handles):
            if q == self.rank:
                areas.append(area)
                continue
            try:
                p = ipc_open(h, dev)
            except Exception as e:  # noqa: BLE001 -- e.g. no P2P / IPC between these GPUs
                err = e
                break
            self._peer_mapped.append(p)
            areas.append(p)
        # Every rank must use the same transport: fall back together.
        ok = torch.tensor([0.0 if err else 1.0],
                          device=self.device if self._nccl else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        if ok.item() < 1.0:
            import warnings
            warnings.warn(f"peer-memory exchange unavailable ({err or 'on another rank'}); "
                          "using the collective transport")
            for p in self._peer_mapped:
                ipc_close(p)
            self._peer_mapped = []
            self.transport = "collective"
            return
        self.state.shard_peer_bind(self.rank, self.world, areas, self.peer_timeout_s)
        self._peer_key = key

    def close(self):
        from .api import ipc_close

        for p in self._peer_mapped:
            ipc_close(p)
        self._peer_mapped = []

    def replay_uploaded_range(self, first: int, count: int):
        """Batches [first, first + count) of the uploaded stream with no host
        round trip between them; their reports. Peer transport: one library
        call per rank (the range is a captured graph); collective transport:
        asynchronous commits with a collective per batch."""
        if self.transport == "peer":
            if self._kind_counts is None:
                raise RuntimeError("upload the stream with ShardedReplay.upload(stream) first")
            ins, dele = self._kind_counts
            self._peer_setup(int(ins[first:first + count].max(initial=0)),
                             int(dele[first:first + count].max(initial=0)))
        if self.transport == "peer":
            self.state.shard_peer_range_begin(first, count)
            return self.state.shard_peer_range_end(count)
        reports = []
        for i, b in enumerate(range(first, first + count)):
            nr, nm = self.state.shard_begin_uploaded(b)
            self._exchange(nr, nm, commit=False)
            if (i + 1) % 256 == 0:  # the pending ring is 256 deep
                reports += self.state.shard_finish()
        return reports + self.state.shard_finish()

    def replay_stream(self, stream):
        """replay(stream) (sparsifier.cpp:550-559) from a host UpdateStream:
        the events are uploaded once (dyg_stream_upload), then the batches
        chain on the device with asynchronous commits and one host
        synchronisation (replay_uploaded_range); the reports."""
        self.upload(stream)
        return self.replay_uploaded_range(0, stream.batch_count)
