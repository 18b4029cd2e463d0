"""Cross-process checkpoint / resume: a session saved after
some batches and loaded in a fresh process replays the rest of the stream
exactly as the uninterrupted reference replay does -- rows, reports and the
update counter (the walker keys, sparsifier.cpp:431, continue from it)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import REPORT_EXACT, same_rows, to_dyg

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_resume_in_fresh_process_matches_uninterrupted_reference(oracle, dyg, tmp_path):
    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(oracle, c)
    ev, nb = s.events(), s.batch_count
    cut = nb // 2 + 1  # inside the decremental half
    ost = oracle.state(g, h, K=c.K, T=c.T, s=c.s, seed=c.walk_seed)
    ref_reports = [ost.replay_batch(s, b) for b in range(nb)]

    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(ev, nb)
    for b in range(cut):
        st.replay_batch(stream, b)
    ckpt = str(tmp_path / "c2.ckpt")
    st.save(ckpt)
    counter = st.update_counter
    st.close()
    np.save(tmp_path / "events.npy", ev)

    # The resume runs in a separate process: nothing but the file carries over.
    script = f"""
import sys, numpy as np
sys.path.insert(0, {REPO!r})
import paper_2505_02741_b200 as D
st = D.SparsifierState.load({ckpt!r})
assert st.update_counter == {counter}, st.update_counter
o = st.options()
assert (o.walk.distortion_threshold, o.walk.step_cap, o.walk.walker_count, o.walk.global_seed, o.batched) == ({c.K!r}, {c.T}, {c.s}, {c.walk_seed}, True), o
stream = D.UpdateStream(np.load({str(tmp_path / 'events.npy')!r}), {nb})
reps = [st.replay_batch(stream, b) for b in range({cut}, {nb})]
np.save({str(tmp_path / 'reports.npy')!r}, np.array([[getattr(r, f) for f in {list(REPORT_EXACT)!r}] for r in reps], dtype=np.float64))
for which, name in ((0, 'g'), (1, 'h')):
    rp, ids, w = st.rows(which)
    np.savez({str(tmp_path)!r} + '/rows_' + name + '.npz', rp=rp, ids=ids, w=w)
print(st.update_counter)
"""
    out = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert int(out.stdout.split()[-1]) == ost.update_counter
    got = np.load(tmp_path / "reports.npy")
    for i, b in enumerate(range(cut, nb)):
        assert [float(ref_reports[b][f]) for f in REPORT_EXACT] == got[i].tolist(), b
    for name, og in (("g", ost.graph()), ("h", ost.sparsifier())):
        z = np.load(tmp_path / f"rows_{name}.npz")
        assert same_rows(og.export(), (z["rp"], z["ids"], z["w"])), name


def test_checkpoint_round_trip_same_process(oracle, dyg, tmp_path):
    c = O.CONFIGS["C1"]
    g, h, s = O.build_config(oracle, c)
    opts = dyg.SparsifierOptions(dyg.WalkConfig(c.K, c.T, c.s, c.walk_seed), True, False)
    st = dyg.SparsifierState(to_dyg(dyg, g), to_dyg(dyg, h), opts)
    stream = dyg.UpdateStream(s.events(), s.batch_count)
    st.replay_batch(stream, 0)
    path = str(tmp_path / "c1.ckpt")
    st.save(path)
    st2 = dyg.SparsifierState.load(path)
    assert st2.update_counter == st.update_counter
    for which in (0, 1):
        assert same_rows(st.rows(which), st2.rows(which))
    for b in range(1, s.batch_count):
        r1, r2 = st.replay_batch(stream, b), st2.replay_batch(stream, b)
        assert [getattr(r1, f) for f in REPORT_EXACT] == [getattr(r2, f) for f in REPORT_EXACT]
    # A flipped byte anywhere fails the checksum.
    raw = bytearray(open(path, "rb").read())
    raw[len(raw) // 2] ^= 0x40
    open(path, "wb").write(bytes(raw))
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState.load(path)
    assert e.value.kind == dyg.ErrorKind.Data
