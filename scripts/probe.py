"""Dev probe: build + solve one config on the GPU with phase timings.
usage: LCN_TIMING=1 python scripts/probe.py c3 [scale]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
t = time.time()
pr = {"c0": configs.config0, "c1": configs.config1, "c3": configs.config3}[which](scale)
print(f"{pr.name} n={pr.n} d={pr.d} buckets={pr.buckets}x{pr.bands} l={pr.landmarks} gen {time.time()-t:.1f}s", flush=True)
ctx = lcn.Context(0)
dp = torch.from_numpy(pr.p.astype(np.float32)).cuda()
dq = torch.from_numpy(pr.q.astype(np.float32)).cuda()
torch.cuda.synchronize()
cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
if os.environ.get("PROBE_SPARSE") == "1":  # the sparse-only operator (KernelOperator::sparse) on the same LSH
    import dataclasses
    pr = dataclasses.replace(pr, landmarks=0)
for _b in range(int(os.environ.get("PROBE_BUILDS", "1")) - 1):  # warm-up builds (pool, first touch)
    if os.environ.get("LCN_TIMING"):
        print(f"---- warm-up build {_b}", file=sys.stderr, flush=True)
    lcn.KernelOperator.from_device(ctx, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost, pr.lam_eff, cfg,
                                   pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
if os.environ.get("LCN_TIMING"):
    print("---- timed build", file=sys.stderr, flush=True)
t = time.time()
op = lcn.KernelOperator.from_device(ctx, dp.data_ptr(), pr.n, dq.data_ptr(), pr.m, pr.d, pr.cost, pr.lam_eff, cfg,
                                    pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
print(f"build {time.time()-t:.2f}s nnz={op.nnz} stored={op.stored} max|delta|={op.max_abs_delta:.3e} cond={op.cond_estimate:.3e}", flush=True)
pm, qm = pr.marginals()
for rep in range(reps):
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False))
    l = pr.landmarks
    B = 8 * op.nnz + 4 * l * (pr.n + pr.m) + 16 * (pr.n + pr.m)
    it_ms = res.device_ms / pr.iters
    print(f"sinkhorn {pr.iters} it: {res.device_ms:.2f} ms ({it_ms:.3f} ms/it, {B/it_ms/1e6:.0f} GB/s algorithmic) "
          f"dist={res.distance/pr.mu:.8f} err={res.marginal_err_final:.3e}", flush=True)
ctx.set_profile(True)
res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False))
ph, it = res.phase_ms()
ctx.set_profile(False)
print("phases ms/it: " + " ".join(f"{k}={v / max(it, 1):.3f}" for k, v in
                                    zip(["col_bands", "col_finalize", "row_bands", "row_finalize"], ph)), flush=True)
