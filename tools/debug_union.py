import sys, os
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from oracle import Oracle, OracleCluster
from paper_2310_00967_b200 import engine
o = Oracle()
for kind in ["stream", "tile"]:
    os.environ["MICRO_K1_KERNEL"] = kind
    n_g, n = 10000, 1
    m = engine.Micro(n_g, n, density=0.01, initial_threshold=0.01)
    ref = OracleCluster(n_g, n, 0.01, 0.01)
    for t in range(3):
        G = np.stack([o.gaussian(7, i, t, n_g) for i in range(n)])
        m.step(list(torch.from_numpy(G).cuda()), 0.01, t)
        r = ref.step(G, 0.01, t)
        idx, sums = m.union()
        st = m.query()
        bad = np.flatnonzero(idx != r["union_idx"])
        print(kind, t, "K", st.K, r["union_idx"].size, "counts", st.counts, r["counts"], "first bad", bad[:5], "nbad", bad.size,
              "tail", idx[-5:], r["union_idx"][-5:])
