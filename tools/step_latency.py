"""Per-step latency of the walk kernels in the thin (latency-bound) regime.

Default: deletion events of H edges on the C5 mesh, 1..N per batch: each
spawns s = 16 recovery walkers on G that mostly run to the step cap T = 100,
so the min-path kernel time / 100 ~ one dependent step (fetch + sample).
REACH=1: insertion events between random vertex pairs with a tiny weight (the
budget never ends a walker), so K1's walkers run on H until a dead end or the
cap; the kernel time / 100 bounds one dependent reach step from above."""
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
REACH = os.environ.get("REACH", "0") == "1"
if REACH:
    n = len(rp) - 1
    for nq in SIZES:
        ev_arr = np.zeros(nq, dtype=D.api.EVENT_DTYPE)
        a = rng.integers(0, n, nq)
        b = (a + n // 2 + rng.integers(0, n // 4, nq)) % n
        ev_arr["kind"] = 0
        ev_arr["u"] = np.minimum(a, b)
        ev_arr["v"] = np.maximum(a, b)
        ev_arr["weight"] = 1e-9
        res = []
        for rep in range(4):  # rep 0 counts steps (instrumented kernel), the rest time the lean one
            st.set_walk_counters(rep == 0)
            st.restore()
            st.reset_stats()
            st.replay_events(ev_arr, None, 0)
            s = st.stats()
            res.append((s["reach_ms"], s["reach_steps"], s["reach_tail_ms"], s["total_ms"]))
        steps = res[0][1]
        rm, _, tail, tot = res[-1]
        print(f"insertions={nq:5d} walkers={S_WALKERS*nq:6d} reach_ms={rm:.4f} tail_ms={tail:.4f} "
              f"steps={steps} mean_steps={steps/(S_WALKERS*nq):.1f} "
              f"us/step(chain<=100)={1000*rm/100:.2f} batch_ms={tot:.4f}", flush=True)
    sys.exit(0)
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
