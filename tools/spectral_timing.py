import time, sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2505_02741_b200 as D
for side in (128, 512):
    g = D.make_mesh(side, side, 1); h = D.build_initial_sparsifier(g, 0.10, 1)
    for it in (1, 5, 30, 60):
        o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-30, max_iterations=it)
        t = time.perf_counter(); e = D.condition_number(g, h, o); dt = time.perf_counter() - t
        print(side*side, it, e.iterations_used, f"{dt:.3f}s", flush=True)
    b = D.random_rhs(side*side, 3)
    for mi in (1, 10, 50):
        t = time.perf_counter(); r = D.pcg_solve(g, b, h, tolerance=1e-30, max_iterations=mi); dt = time.perf_counter() - t
        print("pcg", side*side, mi, r.iterations, f"{dt:.3f}s", flush=True)
