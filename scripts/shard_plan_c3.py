"""Bucket-sharded partition of configs[3] (lcn_shard_plan_*, host only) from
the GPU's bucket ids of both bands (tests/parity_c3_gpu.py dump) ->
profiles/shard_plan_c3.json: owned / halo points and exchange slots per rank
for world 1, 2, 4, 8, and the exchange bytes per half-iteration."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_06876_b200 import ShardPlan  # noqa: E402

src_npz = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "scratch", "parity_c3_gpu.npz")
ids = np.load(src_npz)["ids"].astype(np.uint32)
n = ids.shape[1] // 2
src, tgt = np.ascontiguousarray(ids[:, :n]), np.ascontiguousarray(ids[:, n:])
l, lp = 512, 512
out = {"config": "configs[3]: n=m=1e6, 2 x 4096 k-means LSH (GPU bucket ids, bit-exact vs the reference), l=512",
       "record_doubles": "16 + lp + max_exp per rank per half-iteration (sinkhorn.cu lcn_iteration_shard)",
       "worlds": {}}
for world in (1, 2, 4, 8):
    t0 = time.perf_counter()
    plan = ShardPlan(src, tgt, 4096, l, world)
    dt = time.perf_counter() - t0
    infos = [plan.info(r) for r in range(world)]
    cost = np.array([i["cost"] for i in infos])
    xs, xt = infos[0]["max_exp_s"], infos[0]["max_exp_t"]
    out["worlds"][str(world)] = {
        "plan_s": dt, "groups": infos[0]["groups"], "cost_imbalance": float(cost.max() / cost.mean()),
        "n_own": [i["n_own"] for i in infos], "m_own": [i["m_own"] for i in infos],
        "n_halo": [i["n_halo"] for i in infos], "m_halo": [i["m_halo"] for i in infos],
        "band0_pairs": [i["band0_pairs"] for i in infos], "max_exp_s": xs, "max_exp_t": xt,
        "allgather_bytes_per_rank_per_iteration": 8 * world * ((16 + lp + xs) + (16 + lp + xt)),
    }
json.dump(out, open(os.path.join(ROOT, "profiles", "shard_plan_c3.json"), "w"), indent=1)
print(json.dumps({k: (v["groups"], v["n_halo"], v["allgather_bytes_per_rank_per_iteration"]) for k, v in out["worlds"].items()}))
