"""Where the grounded-Laplacian factorisation's time goes (DYG_SPECTRAL_DEBUG)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DYG_SPECTRAL_DEBUG"] = "1"
import paper_2505_02741_b200 as D
for side in [int(a) for a in sys.argv[1:]] or [512, 1024]:
    g = D.make_mesh(side, side, 1); h = D.build_initial_sparsifier(g, 0.10, 1)
    o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-30, max_iterations=2)
    t = time.perf_counter(); D.condition_number(g, h, o); print(side * side, f"{time.perf_counter() - t:.2f}s", flush=True)
