"""Spectral evaluation timings on the device vs the numpy/scipy restatement
(CPU, oracle/spectral_ref.py) on mesh graphs: kappa (iterative Lanczos) and
PCG with the L_H preconditioner. Usage: python tools/spectral_bench.py [side ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2505_02741_b200 as D
from oracle import spectral_ref as S

for side in [int(a) for a in sys.argv[1:]] or [128, 256, 512]:
    g = D.make_mesh(side, side, 1)
    h = D.build_initial_sparsifier(g, 0.10, 1)
    rg, rh = [tuple(np.asarray(a) for a in x.rows()) for x in (g, h)]
    n = g.vertex_count()
    o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-3, max_iterations=60)
    t = time.perf_counter(); e = D.condition_number(g, h, o); tg = time.perf_counter() - t
    # Warm: the same H again (library initialised, ordering cached), then H
    # after a small edit (a near pattern: the cached ordering is reused).
    t = time.perf_counter(); D.condition_number(g, h, o); tw = time.perf_counter() - t
    print(f"n={n} kappa gpu first call {tg:.2f}s, warm same H {tw:.2f}s", flush=True)
    r, tc = {"kappa": float("nan"), "iterations": 0}, 0.0
    if not os.environ.get("NOCPU"):
        t = time.perf_counter()
        r = S.condition_iterative(S.laplacian(*rg), S.laplacian(*rh), 1e-3, 60)
        tc = time.perf_counter() - t
    print(f"n={n} kappa gpu={e.kappa:.6g} ({e.iterations_used} it, {e.inner_iterations} inner CG it) "
          f"{tg:.2f}s | cpu restatement={r['kappa']:.6g} ({r['iterations']} it) {tc:.2f}s", flush=True)
    b = D.random_rhs(n, 3)
    t = time.perf_counter(); p = D.pcg_solve(g, b, h, tolerance=1e-8); tg = time.perf_counter() - t
    it, rel, tc = 0, float("nan"), 0.0
    if not os.environ.get("NOCPU"):
        t = time.perf_counter()
        x, it, rel, ok, _ = S.pcg_solve(S.laplacian(*rg), b, S.Preconditioner(S.laplacian(*rh)),
                                        1e-8)
        tc = time.perf_counter() - t
    print(f"n={n} pcg gpu {p.iterations} it ({p.inner_iterations} inner) rel={p.relative_residual:.2e} "
          f"{tg:.2f}s | cpu restatement {it} it rel={rel:.2e} {tc:.2f}s", flush=True)
