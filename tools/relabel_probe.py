"""Layout probe: does a locality-preserving vertex numbering speed the walks?

Builds the C5 inputs, then replays them (device-resident, as bench.py's
device step) under the generator's row-major numbering and under a relabeled
copy (Morton or Hilbert order of the mesh coordinates, or a BFS order). The
relabeled problem is isomorphic -- same rows in the same order, ids mapped --
so the walks draw the same samples and do the same steps; only the memory
placement of the rows changes. Prints per-phase device times for each.

Usage: python tools/relabel_probe.py [--config C5] [--order morton|hilbert|bfs] [--steps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def morton(r, c, bits):
    def spread(x):
        x = x.astype(np.uint64)
        out = np.zeros_like(x)
        for b in range(bits):
            out |= ((x >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
        return out
    return spread(r) | (spread(c) << np.uint64(1))


def hilbert(r, c, order):
    x, y = c.astype(np.int64).copy(), r.astype(np.int64).copy()
    d = np.zeros_like(x)
    s = 1 << (order - 1)
    while s > 0:
        rx = (x & s) > 0
        ry = (y & s) > 0
        d += s * s * ((3 * rx) ^ ry)
        # rotate
        flip = ~ry
        sw_x = np.where(flip & rx, s - 1 - x, x)
        sw_y = np.where(flip & rx, s - 1 - y, y)
        x2 = np.where(flip, sw_y, sw_x)
        y2 = np.where(flip, sw_x, sw_y)
        x, y = x2, y2
        s >>= 1
    return d


def bfs_order(rp, ids):
    n = len(rp) - 1
    seen = np.zeros(n, bool)
    order = []
    from collections import deque
    for s in range(n):
        if seen[s]:
            continue
        seen[s] = True
        q = deque([s])
        while q:
            u = q.popleft()
            order.append(u)
            for v in ids[rp[u]:rp[u + 1]]:
                if not seen[v]:
                    seen[v] = True
                    q.append(int(v))
    return np.array(order, np.int64)


def relabel_rows(rows, newid):
    rp, ids, w = (np.asarray(x) for x in rows)
    n = len(rp) - 1
    deg = np.diff(rp.astype(np.int64))
    old_of_new = np.empty(n, np.int64)
    old_of_new[newid] = np.arange(n)
    ndeg = deg[old_of_new]
    nrp = np.zeros(n + 1, np.uint64)
    nrp[1:] = np.cumsum(ndeg)
    # gather each new row from its old row, ids mapped
    starts = rp[old_of_new].astype(np.int64)
    idx = np.repeat(starts - nrp[:-1].astype(np.int64), ndeg) + np.arange(int(nrp[-1]))
    nids = newid[ids[idx].astype(np.int64)].astype(np.uint32)
    nw = w[idx]
    return nrp, nids, nw


def run(D, g_rows, h_rows, events, nb, steps):
    import torch
    g = D.DynamicGraph.from_rows(*g_rows)
    h = D.DynamicGraph.from_rows(*h_rows)
    opts = D.SparsifierOptions(D.WalkConfig(bench.K_BUDGET, bench.T_CAP, bench.WALKERS,
                                            bench.WALK_SEED), True, False)
    st = D.SparsifierState(g, h, opts)
    ts = torch.cuda.Stream()
    torch.cuda.set_stream(ts)
    st.set_stream(ts.cuda_stream)
    st.snapshot()
    stream = D.UpdateStream(events, nb)
    st.upload_stream(stream)
    st.restore()
    first = st.replay_uploaded_range(0, nb)
    st.reset_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ts)
    for _ in range(steps):
        st.restore()
        st.replay_uploaded_range(0, nb)
    e1.record(ts)
    torch.cuda.synchronize()
    s = st.stats()
    out = {"ms_per_step": e0.elapsed_time(e1) / steps,
           "reach_ms": s["reach_ms"] / steps, "reach_tail_ms": s["reach_tail_ms"] / steps,
           "minpath_ms": s["minpath_ms"] / steps, "commit_ms": s["commit_ms"] / steps,
           "prep_ms": s["prep_ms"] / steps,
           "reach_steps": s["reach_steps"] // steps, "minpath_steps": s["minpath_steps"] // steps}
    rep = [(r.insertions_kept, r.paths_recovered, r.walker_steps) for r in first]
    st.close()
    return out, rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--order", default="morton", choices=["morton", "hilbert", "bfs"])
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import paper_2505_02741_b200 as D
    rows, cols, kind, *_ = bench.config_shape(a.config)
    g, h, s = bench.make_inputs_product(a.config)
    g_rows, h_rows = g.rows(), h.rows()
    ev = np.array(s.events, copy=True)
    nb = s.batch_count
    n = len(g_rows[0]) - 1
    v = np.arange(n)
    r, c = v // cols, v % cols
    bits = int(np.ceil(np.log2(max(rows, cols))))
    if a.order == "morton":
        key = morton(r, c, bits)
    elif a.order == "hilbert":
        key = hilbert(r, c, bits)
    else:
        key = np.empty(n, np.int64)
        key[bfs_order(*[np.asarray(x) for x in g_rows[:2]])] = np.arange(n)
    newid = np.empty(n, np.int64)
    newid[np.argsort(key, kind="stable")] = np.arange(n)
    base, rep0 = run(D, g_rows, h_rows, ev, nb, a.steps)
    ev2 = ev.copy()
    ev2["u"] = newid[ev["u"].astype(np.int64)]
    ev2["v"] = newid[ev["v"].astype(np.int64)]
    rel, rep1 = run(D, relabel_rows(g_rows, newid), relabel_rows(h_rows, newid), ev2, nb, a.steps)
    print(json.dumps({"config": a.config, "order": a.order, "row_major": base, "relabeled": rel,
                      "same_reports": rep0 == rep1}))


if __name__ == "__main__":
    main()
