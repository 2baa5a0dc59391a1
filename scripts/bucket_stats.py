"""Dev probe: bucket-shape distribution of the k-means LSH bands for a config
and the per-CTA load of the band kernels' round-robin work split.
usage: python scripts/bucket_stats.py c3 0.5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
pr = {"c0": configs.config0, "c1": configs.config1, "c3": configs.config3}[which](scale)
ctx = lcn.Context(0)
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
ids = lcn.lsh_kmeans_buckets(ctx, pr.p, pr.q, cfg)
n = pr.n
G = 148
for b in range(pr.bands):
    s = np.bincount(ids[b, :n].astype(np.int64), minlength=pr.buckets)
    t = np.bincount(ids[b, n:].astype(np.int64), minlength=pr.buckets)
    ms = (t + 3) & ~3
    area = s * ms
    ok = (s <= 1024) & (t <= 1024) & (s > 0) & (t > 0)
    print(f"band {b}: buckets {pr.buckets} nonempty src {np.count_nonzero(s)} tgt {np.count_nonzero(t)} "
          f"streamable {ok.sum()} oversized {((s > 1024) | (t > 1024)).sum()}")
    for name, v in [("n_b", s), ("m_b", t), ("area", area)]:
        q = np.percentile(v, [0, 10, 50, 90, 99, 100])
        print(f"   {name:5s} pct0/10/50/90/99/100 = " + " ".join(f"{x:.0f}" for x in q))
    w = np.argsort(-area[ok], kind="stable")
    sa, ss = area[ok][w], s[ok][w]
    rows_cta = np.zeros(G); bytes_cta = np.zeros(G)
    for i in range(len(w)):
        rows_cta[i % G] += ss[i]; bytes_cta[i % G] += 4 * sa[i]
    print(f"   round-robin per CTA: rows mean {rows_cta.mean():.0f} max {rows_cta.max():.0f}; "
          f"bytes mean {bytes_cta.mean()/1e6:.2f} MB max {bytes_cta.max()/1e6:.2f} MB")
    narrow = ms[ok] <= 64
    print(f"   rows in buckets with m_b<=64: {s[ok][narrow].sum()} of {s[ok].sum()}; "
          f"area share {area[ok][narrow].sum()/area[ok].sum():.3f}")
