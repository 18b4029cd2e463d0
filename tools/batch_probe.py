"""Per-batch phase split of a device replay (C5 by default): replays the
uploaded stream one batch at a time (same graphs and kernels as a range
replay) after a restore, a few times, and prints per batch kind the mean
device time of each phase from the kernel-written stamps (dyg_stats deltas).

Usage: python tools/batch_probe.py [--config C5] [--reps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402

FIELDS = ("total_ms", "prep_ms", "reach_ms", "reach_tail_ms", "minpath_ms", "minpath_walk_ms",
          "commit_ms", "walk_commit_gap_ms", "batch_gap_ms", "flow_ms_promote", "flow_ms_emit",
          "flow_ms_apply", "flow_ms_reset")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2505_02741_b200 as D
    g, h, s = bench.make_inputs_product(a.config)
    opts = D.SparsifierOptions(D.WalkConfig(bench.K_BUDGET, bench.T_CAP, bench.WALKERS,
                                            bench.WALK_SEED), True, False)
    st = D.SparsifierState(g, h, opts)
    ts = torch.cuda.Stream()
    torch.cuda.set_stream(ts)
    st.set_stream(ts.cuda_stream)
    st.snapshot()
    st.upload_stream(s)
    nb = s.batch_count
    kinds = s.kind_counts()
    per = {f: np.zeros(nb) for f in FIELDS}
    for rep in range(a.reps + 1):
        st.restore()
        for b in range(nb):
            st.reset_stats()
            st.replay_uploaded_range(b, 1)
            x = st.stats()
            if rep:
                for f in FIELDS:
                    per[f][b] += float(x[f]) / a.reps
    out = {"config": a.config, "batches": nb}
    ins = (kinds[0] > 0) & (kinds[1] == 0)
    for name, m in (("insertion", ins), ("deletion", ~ins)):
        out[name] = {f: round(float(per[f][m].mean()) * 1000.0, 2) for f in FIELDS}  # µs per batch
        out[name]["batches"] = int(m.sum())
    print(json.dumps(out))
    st.close()


if __name__ == "__main__":
    main()
