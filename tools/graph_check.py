import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2505_02741_b200 as D
g = D.make_mesh(64, 64, 1); h = D.build_initial_sparsifier(g, 0.1, 1)
s = D.generate_update_stream(g, D.StreamGenOptions(0.25, 0.01, 4, 7, 0))
st = D.SparsifierState(g, h, D.SparsifierOptions(D.WalkConfig(100.0, 100, 16, 42), True, False))
for b in range(s.batch_count):
    st.replay_batch(s, b)
print(st.stats()["graph_launches"], st.stats()["kernel_launches"])
