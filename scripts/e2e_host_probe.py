"""Dev probe: the bench's e2e leg (lcn_op_lcn_lsh from pinned fp64 host
buffers + lcn_sinkhorn) with phase timings (LCN_TIMING=1).
usage: LCN_TIMING=1 python scripts/e2e_host_probe.py [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ.setdefault("LCN_POOL_RESERVE_GB", "64")
import torch
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pr = configs.config3(1.0)
ctx = lcn.Context(0)
pm, qm = pr.marginals()
p64 = torch.from_numpy(pr.p).pin_memory().numpy()
q64 = torch.from_numpy(pr.q).pin_memory().numpy()
pm64 = torch.from_numpy(pm).pin_memory().numpy()
qm64 = torch.from_numpy(qm).pin_memory().numpy()
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False)
for r in range(reps):
    print(f"---- rep {r}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t0 = time.time()
    op = lcn.KernelOperator.lcn_lsh(ctx, p64, q64, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    t1 = time.time()
    res = lcn.sinkhorn(op, pm64, qm64, opts)
    d = res.distance
    t2 = time.time()
    print(f"rep {r}: build {t1 - t0:.3f} s, solve {t2 - t1:.3f} s, total {t2 - t0:.3f} s, distance {d:.8f}",
          file=sys.stderr, flush=True)
    del op, res
