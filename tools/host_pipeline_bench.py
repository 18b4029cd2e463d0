"""SURVEY 8f row 2 evidence: the host input pipeline (update-stream generation
with locality, MatrixMarket round trip) of libdyg vs the reference build
(oracle/_ref, test infrastructure) on the same inputs; checks the outputs are
identical. CPU only. Usage: python tools/host_pipeline_bench.py [side] [L]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2505_02741_b200 as D
from oracle import oracle as O

side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
L = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ref = O.load("reference")
g_ref = ref.make_mesh(side, side, 1)
g = D.DynamicGraph.from_rows(*g_ref.export())
n = g.vertex_count()
t = time.perf_counter()
s_ours = D.generate_update_stream(g, D.StreamGenOptions(0.25, 0.03, 10, 7, L))
t_ours = time.perf_counter() - t
t = time.perf_counter()
s_ref = ref.generate_stream(g_ref, 0.25, 0.03, 10, 7, L)
t_ref = time.perf_counter() - t
same = np.array_equal(np.asarray(s_ours.events).view(np.uint8),
                      np.asarray(s_ref.events()).view(np.uint8))
print(f"generate_update_stream n={n} L={L}: libdyg {t_ours:.2f}s, reference {t_ref:.2f}s, "
      f"identical={same}")
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "g.mtx")
    D.save_matrix_market(g, p)
    t = time.perf_counter(); g2 = D.load_matrix_market(p); t_ours = time.perf_counter() - t
    t = time.perf_counter(); g3 = ref.load_matrix_market(p); t_ref = time.perf_counter() - t
    a, b = g2.rows(), g3.export()
    same = all(np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
               for x, y in zip(a, b))
    print(f"load_matrix_market n={n}: libdyg {t_ours:.2f}s, reference {t_ref:.2f}s, identical={same}")
