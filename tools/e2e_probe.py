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
    print("graph launches", st.stats()["graph_launches"], "kernels", st.stats()["kernel_launches"])
    print(f"rep {rep}: total {tot:.2f} ms, sum wall {sum(walls):.2f}, sum device {sum(devs):.2f}")
for b in range(0):
    print(f"  batch {b:2d}: n={len(batches[b][0]):6d} wall {walls[b]:.3f} ms device {devs[b]:.3f} ms gap {walls[b]-devs[b]:.3f}")
# host-side pieces
ev = batches[0][0]
t = time.perf_counter(); k = int((ev["kind"] == 1).sum()); print("numpy count ms", 1e3 * (time.perf_counter() - t))
# H2D bandwidth of a pinned 2.5 MB buffer and the bare call overhead
import torch
src = torch.empty(2_516_592, dtype=torch.uint8).pin_memory()
dst = torch.empty_like(src, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 20
print(f"H2D 2.5 MB pinned: {dt*1e6:.1f} us ({2.5166/dt/1e3:.1f} GB/s)")
empty = np.zeros(0, D.api.EVENT_DTYPE)
t = time.perf_counter()
for _ in range(200):
    st.replay_events(empty, None, 0)
print(f"empty replay_events call: {(time.perf_counter()-t)/200*1e6:.1f} us")
one = batches[10][0][:1]
t = time.perf_counter()
for _ in range(50):
    try:
        st.replay_events(one, None, 10)
    except Exception:
        pass
print(f"1-event deletion batch call: {(time.perf_counter()-t)/50*1e6:.1f} us")
