"""Generate the committed golden fixtures from the REFERENCE oracle
(oracle/_ref/libdyg_ref.so = /root/reference/proj/src compiled unmodified).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the plain-C restatement and the GPU path on machines where
the reference cannot be rebuilt (the GPU box has no /root/reference).

Contents of golden.npz:
  walker_seeds      walker_seed(g, uid, i) for a grid of inputs (rng.hpp:45-50)
  rb_*              run_batch on make_random_connected(80,120,47), 64 mixed
                    queries, K=20, T=100, s=8, seed=3 (test_walk.cpp:228-260)
  c1_reports        BatchReport of every C1 batch
  c1_g_* / c1_h_*   final C1 rows of G and H (row_ptr, ids, w)
  c2_reports        BatchReport of every C2 batch (10 ins + 10 del)
  c2_g_* / c2_h_*   final C2 rows
  adv_events        a mixed adversarial stream on make_mesh(12,13,1)
  adv_reports       its per-batch reports (K=3, T=12, s=4, seed=1)
  adv_g_* / adv_h_* its final rows
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from tests.test_gpu_replay import adversarial_stream  # noqa: E402


def replay_all(orc, g, h, events, nb, K, T, s, seed):
    st = orc.state(g, h, K=K, T=T, s=s, seed=seed)
    stream = orc.stream(events, nb)
    reps = np.zeros(nb, O.REPORT_DTYPE)
    for b in range(nb):
        reps[b] = st.replay_batch(stream, b)
    reps["wall_ms"] = 0.0
    return reps, st.graph().export(), st.sparsifier().export()


def main():
    orc = O.load("reference")
    out = {}
    seeds = np.zeros((4, 5, 17), np.uint64)
    for a, gs in enumerate([0, 1, 42, 2024]):
        for b, uid in enumerate([0, 1, 7, 1000, 2**40]):
            for i in range(17):
                seeds[a, b, i] = orc.walker_seed(gs, uid, i)
    out["walker_seeds"] = seeds

    g = orc.make_random_connected(80, 120, 47)
    rng = np.random.default_rng(9)
    q = np.zeros(64, O.QUERY_DTYPE)
    for i in range(64):
        p, t = int(rng.integers(80)), int(rng.integers(80))
        if p == t:
            t = (t + 1) % 80
        q[i] = (1 if i % 3 == 0 else 0, p, t, 0, 0.5 + rng.random(), i)
    res, paths = orc.run_batch(g, q, 20.0, 100, 8, 3)
    out["rb_graph_rp"], out["rb_graph_ids"], out["rb_graph_w"] = g.export()
    out["rb_queries"], out["rb_results"], out["rb_paths"] = q, res, paths

    for name in ("C1", "C2"):
        c = O.CONFIGS[name]
        G, H, S = O.build_config(orc, c)
        reps, gr, hr = replay_all(orc, G, H, S.events(), S.batch_count, c.K, c.T, c.s, c.walk_seed)
        key = name.lower()
        out[f"{key}_reports"] = reps
        out[f"{key}_g_rp"], out[f"{key}_g_ids"], out[f"{key}_g_w"] = gr
        out[f"{key}_h_rp"], out[f"{key}_h_ids"], out[f"{key}_h_w"] = hr

    G = orc.make_mesh(12, 13, 1)
    H = orc.build_initial_sparsifier(G, 0.10, 1)
    ev, nb = adversarial_stream(orc, G, 1)
    reps, gr, hr = replay_all(orc, G, H, ev, nb, 3.0, 12, 4, 1)
    out["adv_events"], out["adv_reports"] = ev, reps
    out["adv_g_rp"], out["adv_g_ids"], out["adv_g_w"] = gr
    out["adv_h_rp"], out["adv_h_ids"], out["adv_h_w"] = hr
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
