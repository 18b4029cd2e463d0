import sys, os, json
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import numpy as np, bench, relabel_probe as R
import paper_2505_02741_b200 as D
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
g, h, s = bench.make_inputs_product(cfg)
out, _ = R.run(D, g.rows(), h.rows(), np.array(s.events, copy=True), s.batch_count, 5)
print(json.dumps(out))
