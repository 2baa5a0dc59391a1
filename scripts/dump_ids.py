"""Dev probe: dump the k-means LSH bucket ids of a config (for host-side
layout studies). usage: python scripts/dump_ids.py c3 1.0 out.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

which, scale, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
pr = {"c0": configs.config0, "c1": configs.config1, "c3": configs.config3}[which](scale)
ctx = lcn.Context(0)
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
ids = lcn.lsh_kmeans_buckets(ctx, pr.p, pr.q, cfg)
np.savez_compressed(out, ids=ids, n=pr.n)
print("saved", ids.shape)
