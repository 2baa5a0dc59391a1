"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs the reference's own sources compiled unmodified (oracle/_ref/libref_lcn.so,
built by `make -C oracle ref` from /root/reference; Nystrom restated because
Eigen is absent) on the seeded synthetic inputs of paper_2107_06876_b200.configs
and on the reference generator's own point sets, and writes small fixtures:
bucket ids, SHA-256 digests of the CSR support and log-K bits, distances,
plan samples and k-means results. Re-run only in the build container:

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import RefLib  # noqa: E402
from paper_2107_06876_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
# (scheme, bands, rows, buckets, branching, seed); scheme = LshScheme value
LSH_CASES = [(0, 2, 1, 4, 2, 42), (0, 3, 2, 4, 2, 17), (0, 1, 1, 16, 2, 5), (1, 1, 1, 4, 2, 42),
             (2, 1, 1, 4, 2, 42), (2, 1, 1, 12, 3, 9), (2, 2, 2, 4, 2, 3)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ref = RefLib()
    fixtures = {}
    arrays = {}
    # --- configs (full configs[0]; configs[1], [3] at test scale) ---------------
    for key, pr in [("c0", configs.config0()), ("c1s", configs.config1(0.05)), ("c3s", configs.config3(0.002))]:
        ids = ref.lsh_buckets(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
        pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
        rows, cols = pairs.arrays()
        pm, qm = pr.marginals()
        if pr.landmarks:
            op = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
        else:
            op = ref.op_sparse(pr.p, pr.q, pr.cost, pr.lam_eff, pairs)
        rp, col, logk = op.csr(0)
        res = op.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
        plan = res.sp_vals if pr.landmarks else res.sparse_vals
        idx = np.linspace(0, len(plan) - 1, 64).astype(np.int64)
        arrays[f"{key}_ids"] = ids.astype(np.uint16)
        arrays[f"{key}_plan_idx"] = idx
        arrays[f"{key}_plan"] = plan[idx]
        arrays[f"{key}_log_s"] = res.log_s[:: max(1, pr.n // 64)]
        fixtures[key] = {"name": pr.name, "n": pr.n, "m": pr.m, "nnz": int(len(rows)),
                         "points_sha256": sha(pr.p, pr.q), "lam_eff": pr.lam_eff,
                         "support_sha256": sha(rp, col), "logk_sha256": sha(logk),
                         "distance": res.distance, "distance_over_mu": res.distance / pr.mu,
                         "iters": res.iters, "warnings": res.n_warnings,
                         "plan_sum": float(np.sum(plan)), "marginal_err_final": res.marginal_err_final}
        if pr.landmarks:
            fixtures[key]["distance_lcn"] = res.distance_lcn()
            fixtures[key]["max_abs_delta"] = op.scalar(0)
    # --- k-means (kmeans.cpp) on seeded mixtures ---------------------------------
    r = np.random.default_rng(7)
    for (n, d, k, seed) in [(40, 3, 4, 1), (500, 8, 16, 7), (3000, 16, 37, 11), (64, 2, 60, 5)]:
        means = r.standard_normal((5, d)) * 3
        x = (means[r.integers(0, 5, n)] + r.standard_normal((n, d))).astype(np.float32).astype(np.float64)
        ctr, asg = ref.lloyd(x, k, 10, seed)
        key = f"lloyd_{n}_{d}_{k}_{seed}"
        arrays[key + "_x"] = x
        arrays[key + "_assign"] = asg
        fixtures[key] = {"centroids_sha256": sha(ctr), "pp": ref.kmeans_pp(x, k, seed).tolist()}
    # --- the reference generator's own point sets (generators.cpp:28-42) --------
    for (n, d, seed) in [(6, 3, 1), (5, 3, 2), (4, 2, 11), (3, 2, 12), (8, 3, 22), (8, 3, 23), (12, 2, 1000),
                         (12, 2, 1001), (20, 3, 900), (20, 3, 901), (3, 2, 1100), (3, 2, 1101), (10, 4, 41),
                         (10, 4, 42)]:
        arrays[f"ball_{n}_{d}_{seed}"] = ref.sample_uniform_ball(n, d, seed)
    # --- the other LSH schemes (lsh.cpp:55-143) on the generator's balls ----------
    # (p, q as in test_lsh.cpp "identical seeds give identical pair sets")
    p = ref.sample_uniform_ball(60, 4, 21)
    q = ref.sample_uniform_ball(50, 4, 22)
    arrays["lsh_p"], arrays["lsh_q"] = p, q
    for (scheme, bands, rows, buckets, branching, seed) in LSH_CASES:
        ids = ref.lsh_buckets_cfg(p, q, scheme, bands, rows, buckets, 10, branching, seed)
        key = "lsh_%d_%d_%d_%d_%d_%d" % (scheme, bands, rows, buckets, branching, seed)
        arrays[key + "_ids"] = ids.astype(np.uint32)
        fixtures[key] = {"max_id": int(ids.max())}
        # hierarchical leaves can overshoot buckets_per_fn (branching > 2); the
        # reference's counting sort then indexes past its range
        # (lsh.cpp:197-200), so pairs are pinned only for in-range ids
        if ids.max() < buckets ** rows:
            pr = ref.lsh_pairs_cfg(p, q, scheme, bands, rows, buckets, 10, branching, seed).arrays()
            fixtures[key].update({"pairs_sha256": sha(*pr), "nnz": int(len(pr[0]))})
    for seed in (0, 7, 2024):
        arrays[f"normal_{seed}"] = ref.normal_draws(seed, 33)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(fixtures, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(fixtures), "fixture records")


if __name__ == "__main__":
    main()
