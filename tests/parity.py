"""Shared parity helpers: drive the product (through its C-ABI) and the
oracle on identical inputs and compare bit-for-bit."""
import numpy as np

from oracle import oracle as O

REPORT_EXACT = O.REPORT_EXACT


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def same_rows(a, b):
    """(row_ptr, ids, w) triples equal including weight bit patterns and order."""
    return all(np.array_equal(bits(x), bits(y)) for x, y in zip(a, b))


def first_row_diff(a, b):
    rpa, ia, wa = a
    rpb, ib, wb = b
    n = min(len(rpa), len(rpb)) - 1
    for u in range(n):
        ra = (ia[rpa[u]:rpa[u + 1]].tolist(), wa[rpa[u]:rpa[u + 1]].tolist())
        rb = (ib[rpb[u]:rpb[u + 1]].tolist(), wb[rpb[u]:rpb[u + 1]].tolist())
        if ra != rb:
            return u, ra, rb
    return None


def to_dyg(D, og):
    """Oracle graph -> product DynamicGraph with identical rows."""
    return D.DynamicGraph.from_rows(*og.export())


def to_stream(D, ostream):
    return D.UpdateStream(ostream.events(), ostream.batch_count)


def compare_replay(D, orc, g, h, stream_events, batch_count, K=100.0, T=100, s=16, seed=42,
                   batched=True, freeze=False, batches=None, check_rows_every=1):
    """Replay the same stream on the oracle and on the device; compare every
    batch's report (exact fields), update counter and (periodically) rows."""
    og, oh = g, h
    ost = orc.state(og, oh, K=K, T=T, s=s, seed=seed, batched=batched, freeze=freeze)
    ostream = orc.stream(stream_events, batch_count)
    opts = D.SparsifierOptions(D.WalkConfig(K, T, s, seed), batched, freeze)
    st = D.SparsifierState(to_dyg(D, og), to_dyg(D, oh), opts)
    dstream = D.UpdateStream(stream_events, batch_count)
    out = []
    for b in (range(batch_count) if batches is None else batches):
        oerr = derr = None
        try:
            r1 = ost.replay_batch(ostream, b)
        except O.OracleError as e:
            oerr = e
        try:
            r2 = st.replay_batch(dstream, b)
        except D.Error as e:
            derr = e
        assert (oerr is None) == (derr is None), (b, oerr, derr)
        if oerr is not None:
            assert int(derr.kind) == oerr.kind, (oerr, derr)
            assert str(derr) == oerr.message, (oerr.message, str(derr))
            out.append(("error", b))
            assert st.update_counter == ost.update_counter
            break
        for f in REPORT_EXACT:
            assert r1[f] == getattr(r2, f), (b, f, r1[f], getattr(r2, f))
        assert st.update_counter == ost.update_counter
        if check_rows_every and (b % check_rows_every == 0 or b == batch_count - 1):
            gd, hd = st.rows(0), st.rows(1)
            go, ho = ost.graph().export(), ost.sparsifier().export()
            assert same_rows(go, gd), ("G rows", b, first_row_diff(go, gd))
            assert same_rows(ho, hd), ("H rows", b, first_row_diff(ho, hd))
        out.append(r2)
    st.close()
    return out
