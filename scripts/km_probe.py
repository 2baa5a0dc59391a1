"""Dev probe: k-means++ seeding on configs[3]-shaped points (timing / ncu).
usage: python scripts/km_probe.py [k] [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
pr = configs.config3(scale)
x = np.concatenate([pr.p, pr.q]).astype(np.float32).astype(np.float64)
ctx = lcn.Context(0)
for rep in range(2):
    t = time.time()
    idx = lcn.kmeans_pp_indices(ctx, x, k, seed=123)
    dt = time.time() - t
    print(f"N={x.shape[0]} k={k}: {dt*1e3:.1f} ms ({dt/k*1e6:.1f} us/step) first={idx[:4]}", flush=True)
