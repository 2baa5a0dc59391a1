"""Dev probe: CUPTI kernel timeline (torch.profiler) of one k-means run; prints
busy time vs wall time and the largest idle gaps between our kernels.
usage: python scripts/timeline.py N K [d]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2107_06876_b200 as lcn

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 512
d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
rng = np.random.default_rng(5)
means = rng.standard_normal((1000, d))
x = (means[rng.integers(0, 1000, N)] + 0.5 * rng.standard_normal((N, d))).astype(np.float32).astype(np.float64)
ctx = lcn.Context(0)
lcn.lloyd(ctx, x[:100000], 64, 2, 1)  # warm-up / module load
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    c, a = lcn.lloyd(ctx, x, K, 10, 7)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in ev)
print(f"kernels {len(ev)}  span {(t1 - t0) / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms")
from collections import defaultdict
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    agg[e.name[:60]][0] += 1
    agg[e.name[:60]][1] += (e.time_range.end - e.time_range.start) / 1e3
for n_, (c_, t_) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {n_:60s} {c_:6d} {t_:9.1f} ms")
gaps = []
for a_, b_ in zip(ev, ev[1:]):
    g = b_.time_range.start - a_.time_range.end
    gaps.append((g, a_.name[:40], b_.name[:40]))
gaps.sort(reverse=True)
tot_gap = sum(g for g, _, _ in gaps if g > 0)
print(f"total idle between kernels {tot_gap / 1e3:.1f} ms; largest:")
for g, a_, b_ in gaps[:10]:
    print(f"  {g / 1e3:8.2f} ms after {a_} before {b_}")
gagg = defaultdict(lambda: [0, 0.0])
for g, a_, b_ in gaps:
    if g > 0:
        gagg[b_][0] += 1
        gagg[b_][1] += g / 1e3
print("idle before each kernel kind:")
for n_, (c_, t_) in sorted(gagg.items(), key=lambda x: -x[1][1])[:10]:
    print(f"  {n_:40s} {c_:6d} {t_:9.1f} ms ({t_ / max(c_, 1) * 1e3:.2f} us each)")
