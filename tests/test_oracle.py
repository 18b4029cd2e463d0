"""Pins the CPU oracle (CPU-only tests).

1. The plain-C restatement reproduces the committed golden vectors
   (tests/golden/golden.npz, generated from the reference build by
   tests/golden/make_golden.py) -- runs anywhere, including the GPU box.
2. The restatement equals the compiled reference on fresh inputs (generators,
   run_batch, full replays) whenever oracle/_ref is available.
3. Both oracles pass the reference's own known-answer tests, re-expressed
   from proj/tests/test_walk.cpp (cited per test).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import bits, same_rows

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def oracles():
    out = ["restate"]
    if O.available("reference"):
        out.append("reference")
    return out


@pytest.fixture(params=oracles())
def orc(request, restate):
    return O.load(request.param)


def rows(z, prefix):
    return z[prefix + "_rp"], z[prefix + "_ids"], z[prefix + "_w"]


# ------------------------------------------------------------- golden vectors
def test_walker_seeds_golden(orc, golden):
    seeds = golden["walker_seeds"]
    for a, gs in enumerate([0, 1, 42, 2024]):
        for b, uid in enumerate([0, 1, 7, 1000, 2**40]):
            for i in range(17):
                assert orc.walker_seed(gs, uid, i) == int(seeds[a, b, i])


def test_run_batch_golden(orc, golden):
    rp, ids, w = golden["rb_graph_rp"], golden["rb_graph_ids"], golden["rb_graph_w"]
    g = orc.graph(len(rp) - 1)
    # rebuild with identical row order: the generator is deterministic
    g = orc.make_random_connected(80, 120, 47)
    assert same_rows(g.export(), (rp, ids, w))
    res, paths = orc.run_batch(g, golden["rb_queries"], 20.0, 100, 8, 3)
    assert np.array_equal(bits(res), bits(golden["rb_results"]))
    assert np.array_equal(paths, golden["rb_paths"])


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_replay_golden(orc, golden, name):
    c = O.CONFIGS[name]
    G, H, S = O.build_config(orc, c)
    st = orc.state(G, H, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    key = name.lower()
    for b in range(S.batch_count):
        r = st.replay_batch(S, b)
        for f in O.REPORT_EXACT:
            assert r[f] == golden[f"{key}_reports"][b][f], (name, b, f)
    assert same_rows(st.graph().export(), rows(golden, f"{key}_g"))
    assert same_rows(st.sparsifier().export(), rows(golden, f"{key}_h"))


def test_adversarial_replay_golden(orc, golden):
    G = orc.make_mesh(12, 13, 1)
    H = orc.build_initial_sparsifier(G, 0.10, 1)
    ev = golden["adv_events"]
    nb = len(golden["adv_reports"])
    st = orc.state(G, H, K=3.0, T=12, s=4, seed=1)
    stream = orc.stream(ev, nb)
    for b in range(nb):
        r = st.replay_batch(stream, b)
        for f in O.REPORT_EXACT:
            assert r[f] == golden["adv_reports"][b][f], (b, f)
    assert same_rows(st.graph().export(), rows(golden, "adv_g"))
    assert same_rows(st.sparsifier().export(), rows(golden, "adv_h"))


# ------------------------------------------------- reference known answers
def test_path_walk_known_answers(orc):
    # test_walk.cpp:15-35
    g = orc.make_path(3)
    t = orc.single_walk(g, 0, 2, 1.0, 10.0, 10, 1)
    assert t["terminal"] == 0 and t["acc"] == 2.0 and t["path"] == [0, 1, 2]
    t = orc.single_walk(g, 0, 2, 1.0, 1.5, 10, 1)
    assert t["terminal"] == 1 and t["acc"] == 2.0 and t["steps"] == 2
    t = orc.single_walk(g, 0, 2, 1.0, 100.0, 1, 1)
    assert t["terminal"] == 2 and t["steps"] == 1


def test_dead_end_and_isolated(orc):
    # test_walk.cpp:38-49
    g = orc.graph(4)
    g.insert(0, 1, 1.0)
    g.insert(0, 2, 1.0)
    t = orc.single_walk(g, 1, 3, 1.0, 100.0, 50, 3)
    assert t["terminal"] == 3 and t["path"] == [1, 0, 2]
    with pytest.raises(O.OracleError):
        orc.single_walk(g, 3, 1, 1.0, 100.0, 50, 3)


def test_loop_erasure_vectors(orc):
    # test_walk.cpp:170-177
    assert orc.loop_erase([0, 1, 2, 3, 1, 4]) == [0, 1, 4]
    assert orc.loop_erase([0, 1, 2]) == [0, 1, 2]
    assert orc.loop_erase([0, 1, 2, 3, 2, 4, 1, 5]) == [0, 1, 5]


def test_case_study_golden(orc):
    # test_walk.cpp:213-226 with support/case_study.hpp:16-40
    h_edges = [(25, 20), (20, 21), (21, 22), (22, 17), (17, 16), (16, 15), (15, 14), (14, 13),
               (13, 12), (12, 11), (11, 10), (10, 9), (22, 23), (23, 24), (17, 18), (18, 19),
               (19, 0), (0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 9)]
    g = orc.graph(26)
    for u, v in h_edges + [(24, 25), (16, 21), (3, 7)]:
        g.insert(u, v, 1.0)
    g.delete(16, 17)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (1, 16, 17, 0, 1.0, 0)
    res, paths = orc.run_batch(g, q, 1e18, 100, 32, 2024)
    assert res["reached"][0] == 1
    assert paths[0, : res["path_len"][0]].tolist() == [16, 21, 22, 17]
    assert res["resistance"][0] == 3.0
    # SURVEY.md 8c extra golden on H(0), K=4, s=16, seed 2024.
    h = orc.graph(26)
    for u, v in h_edges:
        h.insert(u, v, 1.0)
    q2 = np.zeros(2, O.QUERY_DTYPE)
    q2[0] = (0, 25, 9, 0, 1.0, 0)
    q2[1] = (0, 25, 17, 0, 1.0, 1)
    res, _ = orc.run_batch(h, q2, 4.0, 100, 16, 2024)
    assert res["reached"][0] == 0
    assert res["reached"][1] == 1 and res["best_estimate"][1] == 4.0


def test_tree_walks_are_exact(orc):
    # test_walk.cpp:65-98: reaching walkers on a tree walk the tree path.
    for seed in range(1, 4):
        t = orc.make_random_connected(30, 0, seed, 0.2, 5.0)
        rp, ids, w = t.export()
        q = []
        for u in range(len(rp) - 1):
            for i in range(rp[u], rp[u + 1]):
                if u < ids[i]:
                    q.append((0, u, int(ids[i]), 0, 1.0, u * 31 + int(ids[i])))
        q = np.array(q, dtype=O.QUERY_DTYPE)
        res, _ = orc.run_batch(t, q, 1e18, 100, 16, 11)
        for k in range(len(q)):
            if res["reached"][k]:
                u, v = int(q["p"][k]), int(q["q"][k])
                assert res["best_estimate"][k] == 1.0 / t.edge_weight(u, v)


def test_monotone_in_walkers(orc):
    # test_walk.cpp:134-150: walkers 0..3 are a prefix of 0..15.
    g = orc.make_random_connected(60, 90, 31)
    q = np.zeros(50, O.QUERY_DTYPE)
    for i in range(50):
        q[i] = (0, 3, 42, 0, 1.0, i)
    a, _ = orc.run_batch(g, q, 1e18, 100, 4, 13)
    b, _ = orc.run_batch(g, q, 1e18, 100, 16, 13)
    for i in range(50):
        if a["reached"][i]:
            assert b["reached"][i] and b["best_estimate"][i] <= a["best_estimate"][i]


# -------------------------------------------- restatement == reference
needs_ref = pytest.mark.skipif(not O.available("reference"),
                               reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("gen", ["mesh", "grid4", "random", "random_pendant"])
def test_restatement_generators_match_reference(restate, reference, gen):
    for seed in (1, 5):
        if gen == "mesh":
            a, b = restate.make_mesh(23, 17, seed), reference.make_mesh(23, 17, seed)
        elif gen == "grid4":
            a, b = restate.make_grid4(19, 21, seed), reference.make_grid4(19, 21, seed)
        else:
            pend = gen == "random_pendant"
            a = restate.make_random_connected(200, 300, seed, 0.1, 10.0, pend)
            b = reference.make_random_connected(200, 300, seed, 0.1, 10.0, pend)
        assert same_rows(a.export(), b.export())
        ha = restate.build_initial_sparsifier(a, 0.1, seed)
        hb = reference.build_initial_sparsifier(b, 0.1, seed)
        assert same_rows(ha.export(), hb.export())
        for loc in (0, 2):
            sa = restate.generate_stream(a, 0.2, 0.05, 4, seed, loc)
            sb = reference.generate_stream(b, 0.2, 0.05, 4, seed, loc)
            assert np.array_equal(bits(sa.events()), bits(sb.events()))
            assert sa.batch_count == sb.batch_count


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("batched,freeze,K", [(True, False, 3.0), (True, True, 10.0),
                                               (True, False, 0.0), (False, False, 5.0)])
def test_restatement_replay_matches_reference(restate, reference, seed, batched, freeze, K):
    from tests.test_gpu_replay import adversarial_stream
    ga = restate.make_mesh(10, 11, seed)
    gb = reference.make_mesh(10, 11, seed)
    ha = restate.build_initial_sparsifier(ga, 0.1, seed)
    hb = reference.build_initial_sparsifier(gb, 0.1, seed)
    ev, nb = adversarial_stream(restate, ga, seed, batches=4, per_batch=40)
    sa = restate.state(ga, ha, K=K, T=20, s=4, seed=seed, batched=batched, freeze=freeze)
    sb = reference.state(gb, hb, K=K, T=20, s=4, seed=seed, batched=batched, freeze=freeze)
    stra, strb = restate.stream(ev, nb), reference.stream(ev, nb)
    for b in range(nb):
        ra, rb = sa.replay_batch(stra, b), sb.replay_batch(strb, b)
        for f in O.REPORT_EXACT:
            assert ra[f] == rb[f], (b, f)
        assert same_rows(sa.graph().export(), sb.graph().export())
        assert same_rows(sa.sparsifier().export(), sb.sparsifier().export())
    assert sa.update_counter == sb.update_counter


@needs_ref
def test_restatement_errors_match_reference(restate, reference):
    for orc_pair in [(restate, reference)]:
        for bad in [(0, 3, 99, 0, 1.0), (0, 4, 4, 0, 1.0), (0, 1, 9, 0, -1.0),
                    (1, 0, 35, 0, 0.0)]:
            msgs = []
            for orc in orc_pair:
                g = orc.make_mesh(6, 6, 1)
                h = orc.build_initial_sparsifier(g, 0.1, 1)
                ev = np.array([(0, 0, 20, 0, 1.0), bad, (0, 2, 30, 0, 1.0)], dtype=O.EVENT_DTYPE)
                st = orc.state(g, h, K=10.0, T=20, s=4, seed=1)
                with pytest.raises(O.OracleError) as e:
                    st.replay_batch(orc.stream(ev, 1), 0)
                msgs.append((e.value.kind, e.value.message, st.update_counter))
            assert msgs[0] == msgs[1]


@pytest.mark.parametrize("batched", [True, False])
def test_reference_decisions_agree_with_reports(reference, batched):
    """oracle/ref/decisions.cpp: the per-event decisions it derives (and pins
    to the reference's own replay -- a divergence raises) add up to every
    batch's counters (sparsifier.cpp:466-533)."""
    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(reference, c)
    st = reference.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed, batched=batched)
    for b in range(s.batch_count):
        r, d = st.replay_batch_decisions(s, b)
        cnt = np.bincount(d, minlength=256)
        assert cnt[0] == r["insertions_kept"] and cnt[1] == r["insertions_pruned"]
        assert cnt[2] + cnt[3] + cnt[4] == r["deletions_seen"]
        assert cnt[3] == r["paths_recovered"] and cnt[4] == r["fallback_activations"]
        assert cnt[255] == 0
