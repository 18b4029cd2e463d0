"""Multi-GPU exchange protocol (paper_2505_02741_b200/parallel.py) on CPU:
world_size 2 (and 3) over gloo at 127.0.0.1. Each rank produces the walk
records of its contiguous query shard (here with the CPU oracle standing in
for the device walk kernels -- test infrastructure only), the records are
all-gathered rank-major exactly as on NVLink, and unpacking must rebuild the
single-process results in query order, bit for bit."""
import os
import socket

import numpy as np
import pytest

from paper_2505_02741_b200.parallel import owner_of, shard_range, slots_per_rank, unpack_records


def test_shard_ranges_partition_queries():
    for nq in [0, 1, 2, 7, 8, 9, 104858]:
        for world in [1, 2, 3, 4, 8]:
            got = []
            for r in range(world):
                lo, hi = shard_range(nq, r, world)
                assert 0 <= hi - lo <= slots_per_rank(nq, world)
                got.extend(range(lo, hi))
            assert got == list(range(nq))
            for q in range(0, nq, max(1, nq // 97)):
                r, i = owner_of(q, nq, world)
                lo, hi = shard_range(nq, r, world)
                assert lo <= q < hi and i == q - lo


REACH_BYTES = 16


def pack_reach(res: np.ndarray, slots: int) -> np.ndarray:
    rec = np.zeros((slots, REACH_BYTES), np.uint8)
    for i in range(len(res)):
        rec[i, 0:4] = np.frombuffer(np.uint32(res["reached"][i]).tobytes(), np.uint8)
        rec[i, 8:16] = np.frombuffer(np.uint64(res["steps_used"][i]).tobytes(), np.uint8)
    return rec


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2505_02741_b200.parallel import allgather_records

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = O.load("restate") if O.available("restate") else O.load("reference")
    g = orc.make_mesh(40, 40, 1)
    h = orc.build_initial_sparsifier(g, 0.1, 1)
    st = orc.generate_stream(g, 0.1, 0.0, 1, 7, 3)
    ev = st.events()
    q = np.zeros(len(ev), O.QUERY_DTYPE)
    q["kind"], q["p"], q["q"] = 0, ev["u"], ev["v"]
    q["w_pq"], q["update_id"] = ev["weight"], np.arange(len(ev))
    nq = len(q)
    lo, hi = shard_range(nq, rank, world)
    res, _ = orc.run_batch(h, q[lo:hi], 100.0, 100, 16, 42)
    local = torch.from_numpy(pack_reach(res, slots_per_rank(nq, world)).reshape(-1))
    gathered = allgather_records(local, world)
    out = unpack_records(gathered.numpy(), nq, world, REACH_BYTES)
    if rank == 0:
        full, _ = orc.run_batch(h, q, 100.0, 100, 16, 42)
        expect = pack_reach(full, nq)
        np.save(result_path, np.array([np.array_equal(out, expect), nq, int(full["reached"].sum())]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allgather_rebuilds_query_order(tmp_path, world):
    import torch.multiprocessing as mp

    path = str(tmp_path / "ok.npy")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    ok, nq, reached = np.load(path)
    assert ok and nq > 100 and 0 < reached < nq
