"""Full-size parity on the benchmark workload (BASELINE.json north star):
the delaunay_n22-shaped C5 stream -- 4.19M vertices, 12.57M edges, 10
incremental + 10 decremental batches, 1,174,323 events -- replayed on the
device and by the CPU reference (all host threads). Every BatchReport
integer field, both densities and every G and H row (ids, weight bits,
order) must match after every batch."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import first_row_diff, same_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c5_full_replay_bit_identical(oracle, dyg):
    os.environ["DYSPARSE_THREADS"] = str(os.cpu_count() or 1)
    c = O.CONFIGS["C5"]
    g, h, s = O.build_config(oracle, c)
    # The product builds its inputs with its own host generators; they must
    # be the reference's, row for row.
    dg = dyg.make_mesh(c.rows, c.cols, c.graph_seed)
    assert same_rows(g.export(), dg.rows())
    dh = dyg.build_initial_sparsifier(dg, c.density, c.h_seed)
    assert same_rows(h.export(), dh.rows())
    ds = dyg.generate_update_stream(dg, dyg.StreamGenOptions(
        c.insert_fraction, c.delete_fraction, c.batches, c.stream_seed, c.locality))
    ev = s.events()
    assert np.array_equal(ev.view(np.uint8), ds.events.view(np.uint8))
    # ... and so is the device stream generator's output.
    gs = dyg.generate_update_stream_gpu(dg, dyg.StreamGenOptions(
        c.insert_fraction, c.delete_fraction, c.batches, c.stream_seed, c.locality))
    assert np.array_equal(ev.view(np.uint8), np.asarray(gs.events).view(np.uint8))

    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    st = dyg.SparsifierState(dg, dh, dyg.SparsifierOptions(
        dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False))
    refs = []
    for b in range(s.batch_count):
        r1 = ost.replay_batch(s, b)
        refs.append(r1)
        r2 = st.replay_batch(ds, b)
        for f in O.REPORT_EXACT:
            assert r1[f] == getattr(r2, f), (b, f, r1[f], getattr(r2, f))
        go, gd = ost.graph().export(), st.rows(0)
        assert same_rows(go, gd), ("G", b, first_row_diff(go, gd))
        ho, hd = ost.sparsifier().export(), st.rows(1)
        assert same_rows(ho, hd), ("H", b, first_row_diff(ho, hd))
    assert st.update_counter == ost.update_counter == len(ev)

    st.close()
    # The same stream as one device-resident range, and through the
    # multi-GPU split's peer-memory exchange (a world of one rank), from
    # fresh sessions: the same reports and the same final G and H.
    nb = s.batch_count
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    for peer in (False, True):
        st = dyg.SparsifierState(dg, dh, opts)
        st.upload_stream(ds)
        if peer:
            ins, dele = ds.kind_counts()
            area, _, _ = st.shard_peer_create(1, int(ins.max()), int(dele.max()))
            st.shard_peer_bind(0, 1, [area])
            st.shard_peer_range_begin(0, nb)
            got = st.shard_peer_range_end(nb)
        else:
            got = st.replay_uploaded_range(0, nb)
        for b in range(nb):
            for f in O.REPORT_EXACT:
                assert refs[b][f] == getattr(got[b], f), (peer, b, f)
        assert same_rows(ost.graph().export(), st.rows(0)), ("G", peer)
        assert same_rows(ost.sparsifier().export(), st.rows(1)), ("H", peer)
        st.close()
