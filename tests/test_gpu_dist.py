"""The multi-GPU split with real processes: world_size 2 over
gloo, both ranks on cuda:0 (this pool has one GPU per box; NCCL refuses two
ranks on one device, so the records are staged through host memory). Each
rank runs the DEVICE protocol -- dyg_shard_begin_uploaded, the walk of its
query range with the device packers (k_pack_*), the all-gather, the device
unpackers (k_unpack_*) and the replicated commit -- and both replicas must
end bit-identical to the single-process reference replay. Both transports:
"peer" (the exchange areas mapped across the two processes with CUDA IPC,
the per-batch epoch handshake in device memory; the two contexts time-slice
the GPU) and "collective" (gloo all-gather through host memory)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, cfg, transport):
    import sys

    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist

    import paper_2505_02741_b200 as D
    from oracle import oracle as O
    from paper_2505_02741_b200.parallel import ShardedReplay

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    orc = O.load("reference" if O.available("reference") else "restate")
    c = O.CONFIGS[cfg]
    g, h, s = O.build_config(orc, c)
    opts = D.SparsifierOptions(D.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    st = D.SparsifierState(D.DynamicGraph.from_rows(*g.export()),
                           D.DynamicGraph.from_rows(*h.export()), opts)
    stream = D.UpdateStream(s.events(), s.batch_count)
    sh = ShardedReplay(st, rank, world, transport=transport, peer_timeout_s=120.0)
    reps = sh.replay_stream(stream)
    torch.cuda.synchronize()
    fields = list(O.REPORT_EXACT)
    np.save(os.path.join(out_dir, f"reports_{rank}.npy"),
            np.array([[float(getattr(r, f)) for f in fields] for r in reps]))
    for which in (0, 1):
        rp, ids, w = st.rows(which)
        np.savez(os.path.join(out_dir, f"rows_{rank}_{which}.npz"), rp=rp, ids=ids, w=w)
    np.save(os.path.join(out_dir, f"bytes_{rank}.npy"), np.array([sh.bytes_exchanged]))
    dist.barrier()  # every rank done reading the others' exchange areas
    sh.close()
    st.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["peer", "collective"])
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_two_processes_device_protocol_match_reference(tmp_path, oracle, cfg, transport):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from tests.parity import same_rows

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), cfg, transport), nprocs=world,
             join=True)
    c = O.CONFIGS[cfg]
    g, h, s = O.build_config(oracle, c)
    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    ref = np.array([[float(r[f]) for f in O.REPORT_EXACT]
                    for r in (ost.replay_batch(s, b) for b in range(s.batch_count))])
    for rank in range(world):
        got = np.load(tmp_path / f"reports_{rank}.npy")
        assert np.array_equal(got, ref), rank
        for which, og in ((0, ost.graph()), (1, ost.sparsifier())):
            z = np.load(tmp_path / f"rows_{rank}_{which}.npz")
            assert same_rows(og.export(), (z["rp"], z["ids"], z["w"])), (rank, which)
        if transport == "collective":  # (the peer transport moves no host-visible buffers)
            assert int(np.load(tmp_path / f"bytes_{rank}.npy")[0]) > 0
