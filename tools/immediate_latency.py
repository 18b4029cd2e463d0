"""Immediate-mode latency: one event at a time through
SparsifierState::apply_insertion / apply_deletion (sparsifier.cpp:243-317),
on the device vs the reference CPU build, on the C5 (or --config) inputs.
Prints one JSON line: per-event latency percentiles and events/s.

Usage: python tools/immediate_latency.py [--config C5] [--ins 2000] [--del 500]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--ins", type=int, default=2000)
    ap.add_argument("--dels", type=int, default=500)
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU build")
    a = ap.parse_args()
    import paper_2505_02741_b200 as D
    g, h, s = bench.make_inputs_product(a.config)
    ev = np.asarray(s.events)
    ins = ev[ev["kind"] == 0][: a.ins]
    dels = ev[ev["kind"] == 1][: a.dels]
    opts = D.SparsifierOptions(D.WalkConfig(bench.K_BUDGET, bench.T_CAP, bench.WALKERS,
                                            bench.WALK_SEED), False, False)
    st = D.SparsifierState(g, h, opts)
    lat = {"insertion": [], "deletion": []}
    for _ in range(20):  # warm-up (graphs, allocations)
        st.apply_insertion(int(ins[0]["u"]), int(ins[0]["v"]), float(ins[0]["weight"]))
        st.apply_deletion(int(ins[0]["u"]), int(ins[0]["v"]))
    for e in ins:
        t = time.perf_counter()
        st.apply_insertion(int(e["u"]), int(e["v"]), float(e["weight"]))
        lat["insertion"].append(time.perf_counter() - t)
    for e in dels:
        t = time.perf_counter()
        st.apply_deletion(int(e["u"]), int(e["v"]))
        lat["deletion"].append(time.perf_counter() - t)
    out = {"config": a.config, "device": {}}
    for k, v in lat.items():
        v = np.asarray(v) * 1e6
        out["device"][k] = {"events": len(v), "p50_us": float(np.percentile(v, 50)),
                            "p99_us": float(np.percentile(v, 99)),
                            "events_per_s": float(len(v) / (v.sum() * 1e-6))}
    if a.cpu:
        from oracle import oracle as O
        orc = O.load("reference" if O.available("reference") else "restate")
        og, oh, _ = bench.make_inputs_oracle(orc, a.config)
        ost = orc.state(og, oh, K=bench.K_BUDGET, T=bench.T_CAP, s=bench.WALKERS,
                        seed=bench.WALK_SEED, batched=False)
        out["cpu_reference"] = {"kind": orc.which}
        for k, sub in (("insertion", ins), ("deletion", dels)):
            x = sub.copy()
            x["batch_index"] = 0
            stream = orc.stream(x, 1)
            t = time.perf_counter()
            ost.replay_batch(stream, 0)  # immediate mode: one event at a time
            dt = time.perf_counter() - t
            out["cpu_reference"][k] = {"events": len(x), "mean_us": 1e6 * dt / len(x),
                                       "events_per_s": len(x) / dt}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
