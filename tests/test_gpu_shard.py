"""The multi-GPU split (dyg_shard_begin / _walk / _commit) driven on ONE GPU:
for world sizes 1, 2, 3 and 8 every rank's walk shard is run in turn into
its slice of a rank-major gathered buffer (exactly the layout the NCCL
all-gather produces), then the replicated commit is applied. Rows and
reports must equal the unsharded replay bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import same_rows, to_dyg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,uploaded", [(1, False), (2, False), (3, False), (8, False),
                                            (1, True), (3, True)])
def test_sharded_replay_equals_single(oracle, dyg, world, uploaded):
    import torch

    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(oracle, c)
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    ref = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    sh = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(s.events(), s.batch_count)
    rb, mb = sh.shard_record_bytes(False), sh.shard_record_bytes(True)
    if uploaded:  # dyg_shard_begin_uploaded: the batch from the device-resident stream
        sh.upload_stream(stream)
    for b in range(s.batch_count):
        r1 = ref.replay_batch(stream, b)
        ev, pos = stream.batch(b)
        nr, nm = sh.shard_begin_uploaded(b) if uploaded else sh.shard_begin(ev, pos, b)
        sr, sm = -(-nr // world), -(-nm // world)
        rall = torch.zeros(max(1, world * sr * rb), dtype=torch.uint8, device="cuda")
        mall = torch.zeros(max(1, world * sm * mb), dtype=torch.uint8, device="cuda")
        for r in range(world):
            sh.shard_walk(r, world, rall.data_ptr() + r * sr * rb, mall.data_ptr() + r * sm * mb)
        torch.cuda.synchronize()
        r2 = sh.shard_commit(world, rall.data_ptr(), mall.data_ptr())
        for f in O.REPORT_EXACT:
            assert getattr(r1, f) == getattr(r2, f), (world, b, f)
    assert same_rows(ref.rows(0), sh.rows(0)) and same_rows(ref.rows(1), sh.rows(1))
    assert ref.update_counter == sh.update_counter


@pytest.mark.parametrize("world", [1, 3])
def test_sharded_async_commits_equal_single(oracle, dyg, world):
    """dyg_shard_commit_async for every batch, one dyg_shard_finish at the end:
    the batches chain on the device (planned update counter and pool
    headroom) and must still equal the unsharded replay bit for bit."""
    import torch

    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(oracle, c)
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    ref = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    sh = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(s.events(), s.batch_count)
    sh.upload_stream(stream)
    rb, mb = sh.shard_record_bytes(False), sh.shard_record_bytes(True)
    keep = []  # record buffers live until the commits have run
    for b in range(s.batch_count):
        nr, nm = sh.shard_begin_uploaded(b)
        sr, sm = -(-nr // world), -(-nm // world)
        rall = torch.zeros(max(1, world * sr * rb), dtype=torch.uint8, device="cuda")
        mall = torch.zeros(max(1, world * sm * mb), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        for r in range(world):
            sh.shard_walk(r, world, rall.data_ptr() + r * sr * rb, mall.data_ptr() + r * sm * mb)
        sh.shard_commit_async(world, rall.data_ptr(), mall.data_ptr())
        keep += [rall, mall]
    reps = sh.shard_finish()
    assert len(reps) == s.batch_count
    for b in range(s.batch_count):
        r1 = ref.replay_batch(stream, b)
        for f in O.REPORT_EXACT:
            assert getattr(r1, f) == getattr(reps[b], f), (world, b, f)
    assert same_rows(ref.rows(0), sh.rows(0)) and same_rows(ref.rows(1), sh.rows(1))
    assert ref.update_counter == sh.update_counter


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_async_stops_at_failing_batch(oracle, dyg, world):
    """A failing batch inside a chain of asynchronous shard commits: the
    device abort flag stops the later batches (already enqueued), and
    dyg_shard_finish reports the reference's error for the failing one."""
    import torch

    g = oracle.make_mesh(9, 9, 3)
    h = oracle.build_initial_sparsifier(g, 0.1, 3)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(0, 0, 40, 0, 1.0), (0, 1, 50, 0, 1.0),            # batch 0: insertions
          (1, edges[0][0], edges[0][1], 1, 0.0),             # batch 1: deletions,
          (1, edges[0][0], edges[0][1], 1, 0.0),             #   the second fails
          (0, 2, 60, 2, 1.0)]                                # batch 2: never commits
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    ost = oracle.state(g, h, K=10.0, T=30, s=8, seed=3)
    ostream = oracle.stream(ev, 3)
    ost.replay_batch(ostream, 0)
    with pytest.raises(O.OracleError) as oe:
        ost.replay_batch(ostream, 1)
    sh = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 3), True, False))
    sh.upload_stream(dyg.UpdateStream(ev, 3))
    rb, mb = sh.shard_record_bytes(False), sh.shard_record_bytes(True)
    keep = []
    for b in range(3):
        nr, nm = sh.shard_begin_uploaded(b)
        sr, sm = -(-nr // world), -(-nm // world)
        rall = torch.zeros(max(1, world * sr * rb), dtype=torch.uint8, device="cuda")
        mall = torch.zeros(max(1, world * sm * mb), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        for r in range(world):
            sh.shard_walk(r, world, rall.data_ptr() + r * sr * rb, mall.data_ptr() + r * sm * mb)
        sh.shard_commit_async(world, rall.data_ptr(), mall.data_ptr())
        keep += [rall, mall]
    with pytest.raises(dyg.Error) as de:
        sh.shard_finish()
    assert str(de.value) == oe.value.message
    assert sh.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), sh.rows(0))
    assert same_rows(ost.sparsifier().export(), sh.rows(1))


def test_async_commits_host_events_and_settled_guard(oracle, dyg):
    """Asynchronous commits of batches begun from HOST event arrays: the
    Python layer keeps every pending batch's buffers alive until
    shard_finish (its error path reads the failing batch's events), and while
    commits are pending every state-reading entry point refuses with a Usage
    error instead of reading stale host-side counters."""
    import gc

    import torch

    g = oracle.make_mesh(9, 9, 3)
    h = oracle.build_initial_sparsifier(g, 0.1, 3)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(0, 0, 40, 0, 1.0), (0, 1, 50, 0, 1.0),
          (1, edges[3][0], edges[3][1], 1, 0.0),
          (1, edges[3][0], edges[3][1], 1, 0.0),             # fails: already deleted
          (0, 2, 60, 2, 1.0)]
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    ost = oracle.state(g, h, K=10.0, T=30, s=8, seed=3)
    ostream = oracle.stream(ev, 3)
    ost.replay_batch(ostream, 0)
    with pytest.raises(O.OracleError) as oe:
        ost.replay_batch(ostream, 1)
    sh = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 3), True, False))
    stream = dyg.UpdateStream(ev, 3)
    rb, mb = sh.shard_record_bytes(False), sh.shard_record_bytes(True)
    keep = []
    for b in range(3):
        bev, bpos = stream.batch(b)
        nr, nm = sh.shard_begin(np.array(bev, copy=True), np.array(bpos, copy=True), b)
        gc.collect()  # the caller's copies are gone; the session's must not be
        rall = torch.zeros(max(1, nr * rb), dtype=torch.uint8, device="cuda")
        mall = torch.zeros(max(1, nm * mb), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        sh.shard_walk(0, 1, rall.data_ptr(), mall.data_ptr())
        sh.shard_commit_async(1, rall.data_ptr(), mall.data_ptr())
        keep += [rall, mall]
    for call in (lambda: sh.rows(0), lambda: sh.replay_batch(stream, 0), sh.snapshot,
                 lambda: sh.apply_insertion(3, 70, 1.0)):
        with pytest.raises(dyg.Error) as ue:
            call()
        assert ue.value.kind == 1 and "dyg_shard_finish" in str(ue.value)
    with pytest.raises(dyg.Error) as de:
        sh.shard_finish()
    assert str(de.value) == oe.value.message
    assert sh.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), sh.rows(0))
    assert same_rows(ost.sparsifier().export(), sh.rows(1))


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_peer_exchange_world1_equals_reference(oracle, dyg, cfg):
    """The peer-memory transport (dyg_shard_peer_*) with a world of one rank:
    prepare, walk, pack into the exchange area, epoch publish / wait, unpack
    and commit as one captured range. Twice (the second replay reuses the
    graph; the epoch keeps advancing on the device), both equal to the
    reference replay; a range larger than the area is refused."""
    c = O.CONFIGS[cfg]
    g, h, s = O.build_config(oracle, c)
    nb = s.batch_count
    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    ref = [ost.replay_batch(s, b) for b in range(nb)]
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    ev = s.events()
    kinds = np.bincount(ev["batch_index"][ev["kind"] == 0].astype(np.int64), minlength=nb)
    kdel = np.bincount(ev["batch_index"][ev["kind"] != 0].astype(np.int64), minlength=nb)
    area, nbytes, handle = st.shard_peer_create(1, int(kinds.max()), int(kdel.max()))
    assert area and nbytes > 0 and len(handle) == 64
    st.shard_peer_bind(0, 1, [area])
    st.upload_stream(dyg.UpdateStream(ev, nb))
    st.snapshot()
    for rep in range(2):
        if rep:
            st.restore()
        st.shard_peer_range_begin(0, nb)
        got = st.shard_peer_range_end(nb)
        assert len(got) == nb
        for b in range(nb):
            for f in O.REPORT_EXACT:
                assert ref[b][f] == getattr(got[b], f), (rep, b, f)
        assert same_rows(ost.graph().export(), st.rows(0))
        assert same_rows(ost.sparsifier().export(), st.rows(1))
    # An area sized below the stream's largest batch refuses the range.
    area2, _, _ = st.shard_peer_create(1, 1, 1)
    st.shard_peer_bind(0, 1, [area2])
    with pytest.raises(dyg.Error) as e:
        st.shard_peer_range_begin(0, nb)
    assert e.value.kind == dyg.ErrorKind.Usage and "exceeds the exchange area" in str(e.value)
    st.close()


def test_sharded_replay_python_paths_world1(oracle, dyg, tmp_path):
    """parallel.ShardedReplay's per-batch entry points in one process (a gloo
    world of one rank): replay_events (host events), replay_uploaded and
    replay_uploaded_range over the collective transport, and
    replay_uploaded_range over the peer transport -- all equal to the
    reference replay."""
    import torch
    import torch.distributed as dist

    from paper_2505_02741_b200.parallel import ShardedReplay

    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(oracle, c)
    nb = s.batch_count
    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    ref = [ost.replay_batch(s, b) for b in range(nb)]
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        torch.cuda.set_stream(torch.cuda.Stream())
        for mode in ("events", "uploaded", "range", "peer"):
            st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
            sh = ShardedReplay(st, 0, 1, transport="peer" if mode == "peer" else "collective")
            stream = dyg.UpdateStream(s.events(), nb)
            if mode == "events":
                got = [sh.replay_events(*stream.batch(b), b) for b in range(nb)]
            else:
                sh.upload(stream)
                if mode == "uploaded":
                    got = [sh.replay_uploaded(b) for b in range(nb)]
                else:
                    got = sh.replay_uploaded_range(0, nb)
            for b in range(nb):
                for f in O.REPORT_EXACT:
                    assert ref[b][f] == getattr(got[b], f), (mode, b, f)
            assert same_rows(ost.graph().export(), st.rows(0)), mode
            assert same_rows(ost.sparsifier().export(), st.rows(1)), mode
            sh.close()
            st.close()
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())
        dist.destroy_process_group()
