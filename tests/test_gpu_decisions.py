"""Per-event keep/drop decisions across the C-ABI (the north star's
"keep/drop decisions must match bit-exactly"; SURVEY.md 8b per_event_decision).

The device returns one DYG_DECISION_* per event (dyg_replay_batch /
_events / _stream / _uploaded_range). The checker is the compiled reference:
oracle/ref/decisions.cpp derives each event's verdict from the reference's
run_batch on the batch-start snapshot and its commit rules
(sparsifier.cpp:220-241, 466-533) and then PINS the derivation to the
reference's own replay_batch (same G and H, bit for bit, or the call fails).
Both sides must agree on every event, including the NONE tail of a failing
batch."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import same_rows, to_dyg
from tests.test_gpu_replay import adversarial_stream

pytestmark = pytest.mark.gpu


def replay_both(dyg, ref, g, h, ev, nb, K=100.0, T=100, s=16, seed=42, batched=True,
                freeze=False, via="batch"):
    """Replay on the reference (with derived decisions) and on the device
    through one of the ABI entry points; compare decisions, reports and rows."""
    ost = ref.state(g, h, K=K, T=T, s=s, seed=seed, batched=batched, freeze=freeze)
    ostream = ref.stream(ev, nb)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h),
                             dyg.SparsifierOptions(dyg.WalkConfig(K, T, s, seed), batched, freeze))
    stream = dyg.UpdateStream(ev, nb)
    o_dec = np.full(len(ev), 255, np.uint8)
    o_err = None
    for b in range(nb):
        sel = np.nonzero(ev["batch_index"] == b)[0]
        try:
            _, d = ost.replay_batch_decisions(ostream, b)
            o_dec[sel] = d
        except O.OracleError as e:
            assert "diverged" not in e.message, e.message
            o_dec[sel] = e.decisions
            o_err = e
            break
    d_dec = np.full(len(ev), 255, np.uint8)
    d_err = None
    try:
        if via == "batch":
            for b in range(nb):
                sel = np.nonzero(ev["batch_index"] == b)[0]
                part = np.full(len(sel), 255, np.uint8)
                try:
                    st.replay_batch(stream, b, decisions=part)
                finally:
                    d_dec[sel] = part
        elif via == "stream":
            st.replay(stream, decisions=d_dec)
        else:
            st.upload_stream(stream)
            st.replay_uploaded_range(0, nb, decisions=d_dec)
    except dyg.Error as e:
        d_err = e
    assert (o_err is None) == (d_err is None), (o_err, d_err)
    if o_err is not None:
        assert str(d_err) == o_err.message
    mism = np.nonzero(o_dec != d_dec)[0]
    assert len(mism) == 0, (len(mism), mism[:10], o_dec[mism[:10]], d_dec[mism[:10]])
    assert same_rows(ost.graph().export(), st.rows(0))
    assert same_rows(ost.sparsifier().export(), st.rows(1))
    st.close()
    return o_dec


@pytest.mark.parametrize("via", ["batch", "stream", "range"])
def test_c2_decisions(reference, dyg, via):
    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(reference, c)
    dec = replay_both(dyg, reference, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                      seed=c.walk_seed, via=via)
    counts = np.bincount(dec, minlength=256)
    assert counts[0] > 0 and counts[1] > 0 and counts[2] > 0 and counts[3] > 0


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("via", ["batch", "stream"])
def test_adversarial_mixed_decisions(reference, dyg, seed, via):
    g = reference.make_mesh(12, 13, seed)
    h = reference.build_initial_sparsifier(g, 0.10, seed)
    ev, nb = adversarial_stream(reference, g, seed)
    replay_both(dyg, reference, g, h, ev, nb, K=3.0, T=12, s=4, seed=seed, via=via)


def test_fallback_heavy_decisions(reference, dyg):
    g = reference.make_random_connected(120, 60, 8)
    h = reference.build_initial_sparsifier(g, 0.0, 8)
    ev, nb = adversarial_stream(reference, g, 8, batches=6, per_batch=40, p_del=0.8)
    dec = replay_both(dyg, reference, g, h, ev, nb, K=4.0, T=3, s=2, seed=8)
    assert (dec == 4).sum() > 0


@pytest.mark.parametrize("freeze,K,batched", [(True, 100.0, True), (False, 0.0, True),
                                              (False, 10.0, False)])
def test_freeze_nofilter_immediate_decisions(reference, dyg, freeze, K, batched):
    g = reference.make_mesh(14, 14, 2)
    h = reference.build_initial_sparsifier(g, 0.10, 2)
    ev, nb = adversarial_stream(reference, g, 2, batches=4, per_batch=30)
    replay_both(dyg, reference, g, h, ev, nb, K=K, T=50, s=8, seed=2, freeze=freeze,
                batched=batched)


@pytest.mark.parametrize("via", ["batch", "stream"])
def test_failing_batch_decisions(reference, dyg, via):
    """An absent deletion mid-batch (sparsifier.cpp:491): the events before it
    have decisions, it and everything after are NONE."""
    g = reference.make_mesh(9, 9, 2)
    h = reference.build_initial_sparsifier(g, 0.1, 2)
    rp, ids, _ = g.export()
    edges = [(u, int(ids[i])) for u in range(len(rp) - 1) for i in range(rp[u], rp[u + 1])
             if u < ids[i]]
    ev = [(0, 0, 40, 0, 1.0), (0, 3, 60, 0, 2.0)]
    ev += [(1, u, v, 1, 0.0) for (u, v) in edges[:12]]
    ev.insert(9, (1, edges[3][0], edges[3][1], 1, 0.0))  # already deleted
    ev.append((0, 5, 70, 2, 1.0))
    ev = np.array(ev, dtype=O.EVENT_DTYPE)
    dec = replay_both(dyg, reference, g, h, ev, 3, K=10.0, T=30, s=8, seed=2, via=via)
    assert (dec[9:] == 255).all() and (dec[:9] != 255).all()


@pytest.mark.slow
def test_c3_decisions(reference, dyg):
    c = O.CONFIGS["C3"]
    g, h, s = O.build_config(reference, c)
    replay_both(dyg, reference, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                seed=c.walk_seed, via="stream")
