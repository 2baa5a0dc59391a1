"""Dev probe: repeated device-resident builds + solves of configs[3] (the bench
e2e loop) with phase timings; PROFILE=1 wraps the first build in a
torch.profiler session like bench.py's kernel trace.
usage: LCN_TIMING=1 python scripts/e2e_probe.py [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pr = configs.config3(1.0)
ctx = lcn.Context(0)
p32 = torch.from_numpy(pr.p.astype(np.float32)).pin_memory()
q32 = torch.from_numpy(pr.q.astype(np.float32)).pin_memory()
pm, qm = pr.marginals()
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False)
for r in range(reps):
    print(f"---- rep {r}", file=sys.stderr, flush=True)
    t = time.time()
    xp, xq = p32.cuda(non_blocking=True), q32.cuda(non_blocking=True)
    torch.cuda.synchronize()
    def build():
        return lcn.KernelOperator.from_device(ctx, xp.data_ptr(), pr.n, xq.data_ptr(), pr.m, pr.d, pr.cost,
                                              pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
    if r == 0 and os.environ.get("PROFILE"):
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            op = build()
    else:
        op = build()
    res = lcn.sinkhorn(op, pm, qm, opts)
    print(f"rep {r}: {time.time() - t:.3f} s dist={res.distance:.8f} free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
    del op, res
