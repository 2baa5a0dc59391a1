"""Dev probe: configs[4] batched LCN timing. usage: python scripts/c4_probe.py [scale]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
t = time.time()
b = configs.config4(scale)
print(f"gen {b.count} problems, rows {b.X.shape[0]}: {time.time()-t:.1f}s", flush=True)
ctx = lcn.Context(0)
for rep in range(3):
    t = time.time()
    dist, st, it = lcn.batched_lcn(ctx, b)
    dt = time.time() - t
    vals, counts = np.unique(st, return_counts=True)
    print(f"batched: {dt*1e3:.1f} ms  {b.count/dt:.0f} problems/s  status {dict(zip(vals.tolist(), counts.tolist()))} "
          f"mean dist {np.nanmean(dist):.4f}", flush=True)
