"""Dev probe: configs[2] dense anchor (n = m = 20000, d = 300, C1's points)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
pr = configs.config1(scale)
ctx = lcn.Context(0, dense_recompute=os.environ.get("LCN_DENSE_RECOMPUTE") == "1")
dp = torch.from_numpy(pr.p.astype(np.float32)).cuda()
dq = torch.from_numpy(pr.q.astype(np.float32)).cuda()
torch.cuda.synchronize()
t = time.time()
op = lcn.KernelOperator.dense_device(ctx, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost, pr.lam_eff)
torch.cuda.synchronize()
print(f"dense n={pr.n} m={pr.m} d={pr.d}: build {time.time() - t:.3f}s", flush=True)
pm, qm = pr.marginals()
for rep in range(int(os.environ.get("PROBE_REPS", "3"))):
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=50, want_plan=False, check_support=False))
    it_ms = res.device_ms / 50
    B = 2 * 4 * pr.n * pr.m
    print(f"50 it: {res.device_ms:.2f} ms ({it_ms:.3f} ms/it, {B / it_ms / 1e6:.0f} GB/s of fp32 log K) "
          f"dist={res.distance:.8f}", flush=True)
