"""Device replay (SparsifierState.replay_batch, sparsifier.cpp:395-559) vs the
CPU oracle: after every batch, every row of G and H (ids and weight bits, in
order), every BatchReport integer field, both densities and the update
counter must be identical. Covers the benchmark configs' shapes and the
adversarial cases the commit engine must get right (coalescing, mixed
batches, re-insertions, set_edge_weight's delete+reinsert, fallbacks,
freeze, K == 0, immediate mode, errors)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import compare_replay, same_rows, to_dyg

pytestmark = pytest.mark.gpu


def cfg_inputs(orc, name):
    c = O.CONFIGS[name]
    g, h, s = O.build_config(orc, c)
    return c, g, h, s


def test_c1_grid_incremental(oracle, dyg):
    c, g, h, s = cfg_inputs(oracle, "C1")
    reps = compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                          seed=c.walk_seed)
    assert len(reps) == 10 and sum(r.insertions_pruned for r in reps) > 0


def test_c2_incremental_then_decremental(oracle, dyg):
    c, g, h, s = cfg_inputs(oracle, "C2")
    reps = compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                          seed=c.walk_seed)
    assert sum(r.paths_recovered for r in reps) > 0


@pytest.mark.slow
def test_c3_delaunay_n18_shape(oracle, dyg):
    c, g, h, s = cfg_inputs(oracle, "C3")
    compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                   seed=c.walk_seed, check_rows_every=5)


def adversarial_stream(orc, g, seed, batches=8, per_batch=60, p_del=0.4, mixed=True,
                       p_existing=0.15, p_reinsert=0.1):
    """Random valid stream: deletions hit live edges (including ones inserted
    earlier in the stream/batch), insertions hit random pairs, existing edges
    (coalesce) and just-deleted edges (re-insert)."""
    rng = np.random.default_rng(seed)
    rp, ids, w = g.export()
    n = len(rp) - 1
    live = {}
    for u in range(n):
        for i in range(rp[u], rp[u + 1]):
            v = int(ids[i])
            if u < v:
                live[(u, v)] = float(w[i])
    deleted = []
    ev = []
    for b in range(batches):
        kind_mode = rng.integers(3) if mixed else (0 if b < batches // 2 else 1)
        for _ in range(per_batch):
            if mixed:
                is_del = rng.random() < p_del
            else:
                is_del = kind_mode == 1
            if is_del and live:
                keys = list(live.keys())
                u, v = keys[rng.integers(len(keys))]
                del live[(u, v)]
                deleted.append((u, v))
                ev.append((1, u, v, b, 0.0))
            else:
                r = rng.random()
                if r < p_existing and live:
                    keys = list(live.keys())
                    u, v = keys[rng.integers(len(keys))]
                elif r < p_existing + p_reinsert and deleted:
                    u, v = deleted[rng.integers(len(deleted))]
                else:
                    u, v = int(rng.integers(n)), int(rng.integers(n))
                    if u == v:
                        continue
                    u, v = min(u, v), max(u, v)
                wt = float(rng.uniform(0.3, 3.0))
                live[(u, v)] = live.get((u, v), 0.0) + wt
                if rng.random() < 0.5:
                    u, v = v, u
                ev.append((0, u, v, b, wt))
    return np.array(ev, dtype=O.EVENT_DTYPE), batches


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("K,T,s", [(100.0, 100, 16), (3.0, 12, 4), (1e18, 40, 3)])
def test_adversarial_mixed_batches(oracle, dyg, seed, K, T, s):
    g = oracle.make_mesh(12, 13, seed)
    h = oracle.build_initial_sparsifier(g, 0.10, seed)
    ev, nb = adversarial_stream(oracle, g, seed)
    compare_replay(dyg, oracle, g, h, ev, nb, K=K, T=T, s=s, seed=seed)


@pytest.mark.parametrize("seed", [5, 6])
def test_adversarial_separate_phases(oracle, dyg, seed):
    g = oracle.make_mesh(16, 16, seed)
    h = oracle.build_initial_sparsifier(g, 0.10, seed)
    ev, nb = adversarial_stream(oracle, g, seed, batches=10, per_batch=80, mixed=False)
    compare_replay(dyg, oracle, g, h, ev, nb, K=5.0, T=30, s=8, seed=seed)


def test_fallback_heavy(oracle, dyg):
    # Tiny T and s: most recovery walks fail, exercising run_local_fallback
    # (sparsifier.cpp:264-280) including H-isolated endpoints.
    g = oracle.make_random_connected(120, 60, 8)
    h = oracle.build_initial_sparsifier(g, 0.0, 8)
    ev, nb = adversarial_stream(oracle, g, 8, batches=6, per_batch=40, p_del=0.8)
    reps = compare_replay(dyg, oracle, g, h, ev, nb, K=4.0, T=3, s=2, seed=8)
    assert sum(r.fallback_activations for r in reps if not isinstance(r, tuple)) > 0


@pytest.mark.parametrize("freeze,K", [(True, 100.0), (False, 0.0)])
def test_freeze_and_no_filter(oracle, dyg, freeze, K):
    g = oracle.make_mesh(14, 14, 2)
    h = oracle.build_initial_sparsifier(g, 0.10, 2)
    ev, nb = adversarial_stream(oracle, g, 2, batches=5)
    compare_replay(dyg, oracle, g, h, ev, nb, K=K, T=50, s=8, seed=2, freeze=freeze)


def test_immediate_mode(oracle, dyg):
    g = oracle.make_mesh(10, 10, 3)
    h = oracle.build_initial_sparsifier(g, 0.10, 3)
    ev, nb = adversarial_stream(oracle, g, 3, batches=3, per_batch=25)
    compare_replay(dyg, oracle, g, h, ev, nb, K=10.0, T=50, s=8, seed=3, batched=False)


def test_heavier_sparsifier_weights_take_delete_reinsert(oracle, dyg):
    # An imported H may carry weights above G's; a coalescing insertion then
    # lowers H's copy via delete + reinsert, moving it to the row ends
    # (set_edge_weight, sparsifier.cpp:207-216).
    g = oracle.make_mesh(8, 8, 4)
    h0 = oracle.build_initial_sparsifier(g, 0.10, 4)
    rp, ids, w = h0.export()
    h = oracle.graph(len(rp) - 1)
    for u in range(len(rp) - 1):
        for i in range(rp[u], rp[u + 1]):
            if u < ids[i]:
                h.insert(u, int(ids[i]), float(w[i]) * 3.0)
    ev = []
    for u in range(len(rp) - 1):
        for i in range(rp[u], rp[u + 1]):
            if u < ids[i] and len(ev) < 40:
                ev.append((0, u, int(ids[i]), 0, 0.25))
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    compare_replay(dyg, oracle, g, h, ev, 1, K=100.0, T=50, s=8, seed=4)


def test_validation_errors_match(oracle, dyg):
    g = oracle.make_mesh(6, 6, 1)
    h = oracle.build_initial_sparsifier(g, 0.1, 1)
    for bad in [(0, 3, 99, 0, 1.0), (0, 4, 4, 0, 1.0), (0, 1, 9, 0, -1.0), (1, 0, 35, 0, 0.0)]:
        ev = np.array([(0, 0, 20, 0, 1.0), bad, (0, 2, 30, 0, 1.0)], dtype=O.EVENT_DTYPE)
        compare_replay(dyg, oracle, g, h, ev, 1, K=10.0, T=20, s=4, seed=1)


def test_absent_deletion_in_deletion_batch_is_exact(oracle, dyg):
    # sparsifier.cpp:491 throws mid-commit; events before it stay applied.
    g = oracle.make_mesh(9, 9, 2)
    h = oracle.build_initial_sparsifier(g, 0.1, 2)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(1, u, v, 0, 0.0) for (u, v) in edges[:12]]
    ev.insert(7, (1, edges[3][0], edges[3][1], 0, 0.0))  # already deleted at event 3
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    ost = oracle.state(g, h, K=10.0, T=30, s=8, seed=2)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 2), True, False))
    with pytest.raises(O.OracleError) as oe:
        ost.replay_batch(oracle.stream(ev, 1), 0)
    with pytest.raises(dyg.Error) as de:
        st.replay_batch(dyg.UpdateStream(ev, 1), 0)
    assert str(de.value) == oe.value.message and int(de.value.kind) == oe.value.kind
    assert st.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))


def test_apply_insertion_and_deletion(oracle, dyg):
    # apply_insertion / apply_deletion (sparsifier.cpp:243-317) == immediate
    # replay, event by event.
    g = oracle.make_mesh(10, 10, 6)
    h = oracle.build_initial_sparsifier(g, 0.1, 6)
    ev, nb = adversarial_stream(oracle, g, 6, batches=1, per_batch=40)
    ost = oracle.state(g, h, K=10.0, T=40, s=8, seed=6, batched=False)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 40, 8, 6), False, False))
    for i, e in enumerate(ev):
        one = np.array([e], dtype=O.EVENT_DTYPE)
        one["batch_index"] = 0
        r1 = ost.replay_batch(oracle.stream(one, 1), 0)
        if e["kind"] == 0:
            d = st.apply_insertion(int(e["u"]), int(e["v"]), float(e["weight"]))
            assert int(d) == (0 if r1["insertions_kept"] else 1)
        else:
            out = st.apply_deletion(int(e["u"]), int(e["v"]))
            expect_kind = (1 if r1["paths_recovered"] else
                           2 if r1["fallback_activations"] else 0)
            assert int(out.kind) == expect_kind
            assert out.edges_added == r1["edges_recovered"]
        assert st.last_event_steps() == r1["walker_steps"]
    assert st.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))


def test_uploaded_stream_and_snapshot_restore(oracle, dyg):
    c, g, h, s = cfg_inputs(oracle, "C2")
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(s.events(), s.batch_count)
    st.snapshot()
    a = [st.replay_batch(stream, b) for b in range(s.batch_count)]
    rows_a = (st.rows(0), st.rows(1))
    st.restore()
    assert st.update_counter == 0
    st.upload_stream(stream)
    st.set_walk_counters(True)  # the instrumented walks: same results, per-step stats
    st.reset_stats()
    b = [st.replay_uploaded(k) for k in range(s.batch_count)]
    for x, y in zip(a, b):
        for f in O.REPORT_EXACT:
            assert getattr(x, f) == getattr(y, f)
    assert same_rows(rows_a[0], st.rows(0)) and same_rows(rows_a[1], st.rows(1))
    stats = st.stats()
    assert stats["kernel_launches"] > 0
    # every walker step is counted once: the reports' total
    assert stats["reach_steps"] + stats["minpath_steps"] == sum(r.walker_steps for r in b)
    assert stats["reach_row_bytes"] >= 32 * stats["reach_steps"] > 0


def test_session_ctor_checks(dyg):
    g = dyg.make_mesh(4, 4, 1)
    h = dyg.DynamicGraph(16)
    h.insert_edge(0, 5, 1.0)  # (0,5) is a diagonal or not an edge of G
    opts = dyg.SparsifierOptions(dyg.WalkConfig(10.0, 100, 16, 0), True, False)
    if g.has_edge(0, 5):
        h = dyg.DynamicGraph(16)
        h.insert_edge(0, 15, 1.0)
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState(g, h, opts)
    assert e.value.kind == dyg.ErrorKind.Data
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState(g, dyg.DynamicGraph(15), opts)
    assert e.value.kind == dyg.ErrorKind.Usage
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState(g, dyg.DynamicGraph(16),
                            dyg.SparsifierOptions(dyg.WalkConfig(10.0, 0, 16, 0), True, False))
    assert e.value.kind == dyg.ErrorKind.Usage


def test_uploaded_range_equals_per_batch(oracle, dyg):
    c, g, h, s = cfg_inputs(oracle, "C2")
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    a = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    b = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(s.events(), s.batch_count)
    ra = [a.replay_batch(stream, k) for k in range(s.batch_count)]
    b.upload_stream(stream)
    rb = b.replay_uploaded_range(0, 7) + b.replay_uploaded_range(7, s.batch_count - 7)
    for x, y in zip(ra, rb):
        for f in O.REPORT_EXACT:
            assert getattr(x, f) == getattr(y, f)
    assert same_rows(a.rows(0), b.rows(0)) and same_rows(a.rows(1), b.rows(1))
    assert a.update_counter == b.update_counter


def test_uploaded_range_stops_at_failing_batch(oracle, dyg):
    g = oracle.make_mesh(9, 9, 3)
    h = oracle.build_initial_sparsifier(g, 0.1, 3)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(0, 0, 40, 0, 1.0), (0, 1, 50, 0, 1.0),            # batch 0: insertions
          (1, edges[0][0], edges[0][1], 1, 0.0),             # batch 1: deletions,
          (1, edges[0][0], edges[0][1], 1, 0.0),             #   the second fails
          (0, 2, 60, 2, 1.0)]                                # batch 2: never runs
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    ost = oracle.state(g, h, K=10.0, T=30, s=8, seed=3)
    ostream = oracle.stream(ev, 3)
    r0 = ost.replay_batch(ostream, 0)
    with pytest.raises(O.OracleError) as oe:
        ost.replay_batch(ostream, 1)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 3), True, False))
    st.upload_stream(dyg.UpdateStream(ev, 3))
    with pytest.raises(dyg.Error) as de:
        st.replay_uploaded_range(0, 3)
    assert str(de.value) == oe.value.message
    assert st.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))
    assert r0["insertions_seen"] == 2


@pytest.mark.parametrize("dup", [False, True])
def test_insertion_fast_path_matches_round_engine(oracle, dyg, monkeypatch, dup):
    # Insertion-only batches of new keys take the sort-based append path;
    # a repeated key in the batch (coalescing inside the batch) must fall
    # back to the dependency rounds. Both must equal the reference.
    g = oracle.make_mesh(20, 20, 5)
    h = oracle.build_initial_sparsifier(g, 0.1, 5)
    st = oracle.generate_stream(g, 0.3, 0.0, 3, 9, 2)
    ev = st.events()
    if dup:  # repeat an earlier key (reversed endpoints) later in batch 0
        e0 = ev[0].copy()
        e0["u"], e0["v"] = ev[0]["v"], ev[0]["u"]
        ev = np.concatenate([ev[:5], [e0], ev[5:]]).astype(O.EVENT_DTYPE)
    compare_replay(dyg, oracle, g, h, ev, st.batch_count, K=100.0, T=100, s=16, seed=9)
    monkeypatch.setenv("DYG_NO_FASTPATH", "1")
    compare_replay(dyg, oracle, g, h, ev, st.batch_count, K=100.0, T=100, s=16, seed=9)


def _replay_all_reference(oracle, g, h, ev, nb, K, T, s, seed):
    ost = oracle.state(g, h, K=K, T=T, s=s, seed=seed)
    ostream = oracle.stream(ev, nb)
    return ost, [ost.replay_batch(ostream, b) for b in range(nb)]


@pytest.mark.parametrize("shuffle", [False, True])
def test_replay_stream_pipelined_equals_reference(oracle, dyg, shuffle):
    # replay(stream) in one call (dyg_replay_stream: uploads pipelined with the
    # batches) must equal the reference's replay batch by batch; a stream whose
    # events are not grouped by batch takes the per-batch path.
    c, g, h, s = cfg_inputs(oracle, "C2")
    ev = s.events()
    if shuffle:
        ev = ev[np.random.default_rng(3).permutation(len(ev))]
        ev = ev[np.argsort(ev["batch_index"], kind="stable")][::-1].copy()
    ost, refs = _replay_all_reference(oracle, g, h, ev, s.batch_count, 100.0, 100, 16, 42)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(100.0, 100, 16, 42), True, False))
    stream = dyg.UpdateStream(ev, s.batch_count)
    assert (stream.batch_offsets() is None) == shuffle
    rep = st.replay(stream)
    assert len(rep.batches) == s.batch_count
    for r1, r2 in zip(refs, rep.batches):
        for f in O.REPORT_EXACT:
            assert r1[f] == getattr(r2, f), (f, r1[f], getattr(r2, f))
    assert st.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))


def test_replay_stream_stops_at_failing_batch(oracle, dyg):
    g = oracle.make_mesh(9, 9, 3)
    h = oracle.build_initial_sparsifier(g, 0.1, 3)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(0, 0, 40, 0, 1.0), (0, 1, 50, 0, 1.0),
          (1, edges[0][0], edges[0][1], 1, 0.0),
          (1, edges[0][0], edges[0][1], 1, 0.0),             # fails
          (0, 2, 60, 2, 1.0)]                                # never runs
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    ost = oracle.state(g, h, K=10.0, T=30, s=8, seed=3)
    ostream = oracle.stream(ev, 3)
    ost.replay_batch(ostream, 0)
    with pytest.raises(O.OracleError) as oe:
        ost.replay_batch(ostream, 1)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 3), True, False))
    with pytest.raises(dyg.Error) as de:
        st.replay(dyg.UpdateStream(ev, 3))
    assert str(de.value) == oe.value.message
    assert st.update_counter == ost.update_counter
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))
    # The session stays usable: the next replay continues from this state.
    st2 = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                              dyg.SparsifierOptions(dyg.WalkConfig(10.0, 30, 8, 3), True, False))
    st2.replay(dyg.UpdateStream(ev[:2], 1))
    assert st2.update_counter == 2


def test_uploaded_stream_with_empty_batches(oracle, dyg):
    """A grouped stream with empty batches (batch 1 and the last) through the
    asynchronous per-batch upload: the uploaded range, the peer-exchange
    range (world 1) and the per-batch reference replay agree."""
    c, g, h, s = cfg_inputs(oracle, "C1")
    ev = s.events().copy()
    nb0 = s.batch_count
    ev["batch_index"] = np.where(ev["batch_index"] >= 1, ev["batch_index"] + 1, 0)
    nb = nb0 + 2  # batch 1 and batch nb - 1 are empty
    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    ostream = oracle.stream(ev, nb)
    ref = [ost.replay_batch(ostream, b) for b in range(nb)]
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    for peer in (False, True):
        st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
        stream = dyg.UpdateStream(ev, nb)
        st.upload_stream(stream)
        if peer:
            ins, dele = stream.kind_counts()
            area, _, _ = st.shard_peer_create(1, int(ins.max()), int(dele.max()))
            st.shard_peer_bind(0, 1, [area])
            st.shard_peer_range_begin(0, nb)
            got = st.shard_peer_range_end(nb)
        else:
            got = st.replay_uploaded_range(0, nb)
        assert [r.batch_index for r in got] == list(range(nb))
        for b in range(nb):
            for f in O.REPORT_EXACT:
                assert ref[b][f] == getattr(got[b], f), (peer, b, f)
        assert same_rows(ost.graph().export(), st.rows(0))
        assert same_rows(ost.sparsifier().export(), st.rows(1))
        assert st.update_counter == ost.update_counter
        st.close()
