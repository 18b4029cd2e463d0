"""Per-step latency of the walk kernels in the thin (latency-bound) regime.

Deletion events of H edges on the C5 mesh, 1..N per batch: each spawns
s = 16 recovery walkers on G that mostly run to the step cap T = 100, so the
min-path kernel time / 100 ~ one dependent step (fetch + sample)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_02741_b200 as D

g = D.make_mesh(2048, 2048, 1)
h = D.build_initial_sparsifier(g, 0.10, 1)
rp, ids, w = h.rows()
rng = np.random.default_rng(1)
# H edges (u < v)
us = np.repeat(np.arange(len(rp) - 1, dtype=np.uint32), np.diff(rp).astype(np.int64))
m = us < ids
eu, ev = us[m], ids[m]
S_WALKERS = int(os.environ.get("SW", "16"))
opts = D.SparsifierOptions(D.WalkConfig(100.0, 100, S_WALKERS, 42), True, False)
st = D.SparsifierState(g, h, opts)
st.snapshot()
SIZES = [int(x) for x in sys.argv[1:]] or [1, 8, 64, 512, 4096]
for nq in SIZES:
    sel = rng.choice(len(eu), nq, replace=False)
    ev_arr = np.zeros(nq, dtype=D.api.EVENT_DTYPE)
    for k, i in enumerate(sel):
        ev_arr[k]["kind"] = 1
        ev_arr[k]["u"] = eu[i]
        ev_arr[k]["v"] = ev[i]
    res = []
    for rep in range(4):
        st.restore()
        st.reset_stats()
        st.replay_events(ev_arr, None, 0)
        s = st.stats()
        res.append((s["minpath_ms"], s["minpath_steps"], s["minpath_tail_ms"], s["commit_ms"], s["total_ms"]))
    mp, steps, tail, cm, tot = res[-1]
    print(f"deletions={nq:5d} walkers={S_WALKERS*nq:6d} minpath_ms={mp:.4f} steps={steps} "
          f"us/step(max chain 100)={1000*mp/100:.2f} commit_ms={cm:.4f} batch_ms={tot:.4f}", flush=True)
