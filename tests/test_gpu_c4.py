"""Full-size parity on the G3_circuit-shaped config (BASELINE.json configs[3],
SURVEY.md 8d C4): grid4(1225, 1225, 1) -- 1.5M vertices, 3.0M edges, a
4-neighbour grid with no diagonals -- H0 = build_initial_sparsifier(0.10, 1)
and 10 insertion batches (insert fraction 0.25, L = 0, stream seed 7) that
grow H towards ~35 % density. Replayed on the device and by the CPU
reference (all host threads): every BatchReport integer field, both
densities and every G / H row (ids, weight bits, order) after EVERY batch.

Also here: K = 10 on C3 (SURVEY.md 8d lists K = 10 beside K = 100; the
budget then ends ~11-13 % of the insertion walkers) and the engine-knob
matrix at C3 scale (each knob forces a path production takes in other
situations: mixed batches, overflowing record buffers, absent deletions)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import compare_replay, first_row_diff, same_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c4_full_replay_bit_identical(oracle, dyg):
    os.environ["DYSPARSE_THREADS"] = str(os.cpu_count() or 1)
    c = O.CONFIGS["C4"]
    g, h, s = O.build_config(oracle, c)
    # The product's own host generators and device initial-sparsifier builder
    # must produce the reference's inputs row for row.
    dg = dyg.make_grid4(c.rows, c.cols, c.graph_seed)
    assert same_rows(g.export(), dg.rows())
    dh = dyg.build_initial_sparsifier_gpu(dg, c.density, c.h_seed)
    assert same_rows(h.export(), dh.rows())
    ds = dyg.generate_update_stream(dg, dyg.StreamGenOptions(
        c.insert_fraction, c.delete_fraction, c.batches, c.stream_seed, c.locality))
    ev = s.events()
    assert np.array_equal(ev.view(np.uint8), ds.events.view(np.uint8))
    assert s.batch_count == 10 and (ev["kind"] == 0).all()

    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    st = dyg.SparsifierState(dg, dh, dyg.SparsifierOptions(
        dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False))
    for b in range(s.batch_count):
        r1 = ost.replay_batch(s, b)
        r2 = st.replay_batch(ds, b)
        for f in O.REPORT_EXACT:
            assert r1[f] == getattr(r2, f), (b, f, r1[f], getattr(r2, f))
        go, gd = ost.graph().export(), st.rows(0)
        assert same_rows(go, gd), ("G", b, first_row_diff(go, gd))
        ho, hd = ost.sparsifier().export(), st.rows(1)
        assert same_rows(ho, hd), ("H", b, first_row_diff(ho, hd))
    assert st.update_counter == ost.update_counter == len(ev)
    # H grows from ~10 % off-tree density towards the paper's ~34 %.
    assert r2.density_sparsifier > 0.3


def test_c3_k10(oracle, dyg):
    c = O.CONFIGS["C3"]
    g, h, s = O.build_config(oracle, c)
    reps = compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=10.0, T=c.T, s=c.s,
                          seed=c.walk_seed, check_rows_every=2)
    assert sum(r.insertions_pruned for r in reps) > 0


@pytest.mark.parametrize("knobs", [
    {"DYG_SINGLE_PASS": "0", "DYG_SHADOW_ROUNDS": "1", "DYG_COMMIT_ROUNDS": "1",
     "DYG_GRAPHS": "0"},
    {"DYG_NO_FASTPATH": "1", "DYG_KEEP_SHADOW": "0", "DYG_FLOW_BALANCE": "0",
     "DYG_REACH_SPLIT": "0"},
    {"DYG_FLOW_CAP": "256"},
], ids=["chain+rounds+eager", "roundsfast+undo+static+slotorder", "flow-overflow"])
def test_c3_engines(oracle, dyg, monkeypatch, knobs):
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    c = O.CONFIGS["C3"]
    g, h, s = O.build_config(oracle, c)
    compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                   seed=c.walk_seed, check_rows_every=5)
