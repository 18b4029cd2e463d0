"""Where the end-to-end time goes: per-batch wall time of replay_events
(host buffers) vs the device time of the same batch (C5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_02741_b200 as D
from paper_2505_02741_b200 import _lib

g = D.make_mesh(2048, 2048, 1)
h = D.build_initial_sparsifier(g, 0.10, 1)
s = D.generate_update_stream(g, D.StreamGenOptions(0.25, 0.01, 10, 7, 0))
print("events base:", type(s.events.base).__name__)
opts = D.SparsifierOptions(D.WalkConfig(100.0, 100, 16, 42), True, False)
st = D.SparsifierState(g, h, opts)
st.snapshot()
batches = [s.batch(b) for b in range(s.batch_count)]
print("batch view pinned-backed:", type(batches[0][0].base).__name__)
for rep in range(3):
    st.restore()
    st.reset_stats()
    walls, devs = [], []
    t_all = time.perf_counter()
    for b, (ev, pos) in enumerate(batches):
        before = st.stats()["total_ms"]
        t = time.perf_counter()
        st.replay_events(ev, pos, b)
        walls.append(1e3 * (time.perf_counter() - t))
        devs.append(st.stats()["total_ms"] - before)
    tot = 1e3 * (time.perf_counter() - t_all)
    print(f"rep {rep}: total {tot:.2f} ms, sum wall {sum(walls):.2f}, sum device {sum(devs):.2f}")
for b in range(len(walls)):
    print(f"  batch {b:2d}: n={len(batches[b][0]):6d} wall {walls[b]:.3f} ms device {devs[b]:.3f} ms gap {walls[b]-devs[b]:.3f}")
# host-side pieces
ev = batches[0][0]
t = time.perf_counter(); k = int((ev["kind"] == 1).sum()); print("numpy count ms", 1e3 * (time.perf_counter() - t))
