"""Initial sparsifier at C5 scale: host pipeline vs device builder (time, equality)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_02741_b200 as D

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g = D.make_mesh(rows, rows, 1)
t = time.perf_counter(); hh = D.build_initial_sparsifier(g, 0.10, 1); th = time.perf_counter() - t
D.build_initial_sparsifier_gpu(g, 0.10, 1)  # warm (context, allocator)
t = time.perf_counter(); hd = D.build_initial_sparsifier_gpu(g, 0.10, 1); td = time.perf_counter() - t
a, b = hh.rows(), hd.rows()
same = all(np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)) for x, y in zip(a, b))
print(f"mesh {rows}x{rows}: n={g.vertex_count()} m={g.edge_count()} |H|={hh.edge_count()} "
      f"host {th:.2f} s, device {td:.3f} s ({th/td:.0f}x), identical={same}")
