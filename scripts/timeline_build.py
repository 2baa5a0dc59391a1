"""Dev probe: CUPTI timeline of the full configs[3] operator build (scale arg)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
pr = configs.config3(scale)
ctx = lcn.Context(0)
dp = torch.from_numpy(pr.p.astype(np.float32)).cuda()
dq = torch.from_numpy(pr.q.astype(np.float32)).cuda()
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    op = lcn.KernelOperator.from_device(ctx, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost, pr.lam_eff, cfg,
                                        pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in ev)
print(f"kernels {len(ev)}  span {(t1 - t0) / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms")
from collections import defaultdict
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    agg[e.name[:70]][0] += 1
    agg[e.name[:70]][1] += (e.time_range.end - e.time_range.start) / 1e3
for n_, (c_, t_) in sorted(agg.items(), key=lambda x: -x[1][1])[:22]:
    print(f"  {n_:70s} {c_:6d} {t_:9.1f} ms")
gaps = []
for a_, b_ in zip(ev, ev[1:]):
    g = b_.time_range.start - a_.time_range.end
    gaps.append((g, a_.name[:45], b_.name[:45]))
gaps.sort(reverse=True)
print(f"total idle between kernels {sum(g for g, _, _ in gaps if g > 0) / 1e3:.1f} ms; largest:")
for g, a_, b_ in gaps[:12]:
    print(f"  {g / 1e3:8.2f} ms after {a_} before {b_}")
import subprocess
print("---- build.cu / capi.cu kernels ----")
for e in ev:
    if "build_cu" in e.name or "capi_cu" in e.name:
        nm = e.name
        core = nm[nm.find("_ZN"):] if "_ZN" in nm else nm
        try:
            dem = subprocess.run(["c++filt", core.split("(")[0]], capture_output=True, text=True).stdout.strip()
        except Exception:
            dem = core
        print(f"  {(e.time_range.end - e.time_range.start) / 1e3:9.2f} ms  {dem[:110]}")
