"""The reference runner's experiment loop over the GPU path (SURVEY.md §8(f)
row 3): `lcn_ot run` configs (config_from_json, runner.cpp:92-141) select
the B200 operators for the `full`, `sparse`, `nystrom` and `lcn` variants.

Mirrors runner.cpp: problems from the seeded generators or LCNPTS1 / text
files (make_problem, :180-204), the degree-based LSH bucket count
(lsh_bucket_count, :206-216), one record per (variant, seed) with the
reference's JSON keys (record_to_json, :143-166), the dense full-Sinkhorn
reference when n m <= 10^6 for rel-err-d, PCC and top-0.1% IoU
(compare_plans, metrics.cpp:21-70), and the CSV / JSON outputs
(write_outputs, :420-445). Every operator and solve runs through the C-ABI on
the GPU; plans are densified and compared on the device. Records run in
order on one context (the reference's worker pool shares its CPU cores; here
the variants share one GPU). `bp` configs run the BP-extended solve
(KernelOperator::with_bp) with the scalar deletion cost on both sides.
"""
from __future__ import annotations

import dataclasses
import json
import math
import sys
import time
from typing import Optional

import numpy as np

from . import native as N

_COSTS = {"euclidean": N.EUCLIDEAN, "negative-dot": N.NEGATIVE_DOT, "cosine-derived": N.COSINE_DERIVED}
_SCHEMES = {"cross-polytope": N.LSH_CROSS_POLYTOPE, "kmeans": N.LSH_KMEANS,
            "hierarchical-kmeans": N.LSH_HIERARCHICAL_KMEANS}
_LANDMARKS = {"kmeans": N.LANDMARK_KMEANS, "kmeans++-sampling": N.LANDMARK_KMEANSPP, "kmeanspp": N.LANDMARK_KMEANSPP}
_MASK = (1 << 64) - 1


@dataclasses.dataclass
class RunConfig:
    """RunConfig / ProblemSpec (runner.hpp), reference defaults."""
    generator: str = "uniform-ball"
    n: int = 100
    m: int = 0
    d: int = 16
    c: int = 4
    D: float = 10.0
    r: float = 0.5
    path_p: str = ""
    path_q: str = ""
    variants: list = dataclasses.field(default_factory=lambda: ["full"])
    cost: str = "euclidean"
    lam: float = 0.05
    neighbors: int = 20
    landmarks: int = 20
    lsh_scheme: str = "kmeans"
    bands: int = 1
    rows_per_band: int = 1
    buckets_per_fn: int = 2  # LshConfig default (lsh.hpp:25); a config's "lsh" object defaults it to 0
    kmeans_iters: int = 10
    branching: int = 2
    bp: bool = False
    deletion_cost: float = 0.0
    landmark_method: str = "kmeans"
    heads: int = 1
    tol: float = -1.0
    max_iters: int = 500
    seeds: list = dataclasses.field(default_factory=lambda: [1])
    output: str = ""
    strict_deterministic: bool = False


def config_from_json(j: dict) -> RunConfig:
    """config_from_json (runner.cpp:92-141)."""
    c = RunConfig()
    pr = j["problem"]
    c.generator = pr["generator"]
    if c.generator == "uniform-ball":
        c.n, c.m, c.d = int(pr["n"]), int(pr.get("m", 0)), int(pr["d"])
    elif c.generator == "clustered":
        c.n, c.d, c.c, c.D, c.r = int(pr["n"]), int(pr["d"]), int(pr["c"]), float(pr["D"]), float(pr["r"])
    elif c.generator == "file":
        c.path_p, c.path_q = pr["p"], pr["q"]
    else:
        raise N.InvalidArgument(f"unknown problem generator '{c.generator}'")
    if "variants" in j:
        c.variants = list(j["variants"])
    if "cost" in j:
        if j["cost"] not in _COSTS:
            raise N.InvalidArgument(f"unknown cost function '{j['cost']}'")
        c.cost = j["cost"]
    c.lam = float(j.get("lambda", 0.05))
    if "budget" in j:
        c.neighbors = int(j["budget"].get("neighbors", 20))
        c.landmarks = int(j["budget"].get("landmarks", 20))
    if "lsh" in j:
        lsh = j["lsh"]
        if "scheme" in lsh:
            if lsh["scheme"] not in _SCHEMES:
                raise N.InvalidArgument(f"unknown LSH scheme '{lsh['scheme']}'")
            c.lsh_scheme = lsh["scheme"]
        c.bands = int(lsh.get("bands", 1))
        c.rows_per_band = int(lsh.get("rows-per-band", 1))
        c.buckets_per_fn = int(lsh.get("buckets-per-fn", 0))
        c.kmeans_iters = int(lsh.get("kmeans-iters", 10))
        c.branching = int(lsh.get("branching", 2))
    if "bp" in j:
        c.bp = bool(j["bp"].get("enabled", False))
        c.deletion_cost = float(j["bp"].get("deletion-cost", 0.0))
    if "landmark-method" in j:
        if j["landmark-method"] not in _LANDMARKS:
            raise N.InvalidArgument(f"unknown landmark method '{j['landmark-method']}'")
        c.landmark_method = j["landmark-method"]
    c.heads = int(j.get("heads", 1))
    c.tol = float(j.get("tol", -1.0))
    c.max_iters = int(j.get("max-iters", 500))
    if "seeds" in j:
        c.seeds = [int(s) for s in j["seeds"]]
    c.output = j.get("output", "")
    c.strict_deterministic = bool(j.get("strict-deterministic", False))
    return c


def config_to_json(c: RunConfig) -> dict:
    """config_to_json (runner.cpp:47-90)."""
    if c.generator == "uniform-ball":
        problem = {"generator": c.generator, "n": c.n, "m": c.m, "d": c.d}
    elif c.generator == "clustered":
        problem = {"generator": c.generator, "n": c.n, "d": c.d, "c": c.c, "D": c.D, "r": c.r}
    else:
        problem = {"generator": c.generator, "p": c.path_p, "q": c.path_q}
    return {"problem": problem, "variants": c.variants, "cost": c.cost, "lambda": c.lam,
            "budget": {"neighbors": c.neighbors, "landmarks": c.landmarks},
            "lsh": {"scheme": c.lsh_scheme, "bands": c.bands, "rows-per-band": c.rows_per_band,
                    "buckets-per-fn": c.buckets_per_fn, "kmeans-iters": c.kmeans_iters, "branching": c.branching},
            "bp": {"enabled": c.bp, "deletion-cost": c.deletion_cost}, "landmark-method": c.landmark_method,
            "heads": c.heads, "tol": c.tol, "max-iters": c.max_iters, "seeds": c.seeds, "output": c.output,
            "strict-deterministic": c.strict_deterministic}


def mix_seed(seed: int, salt: int) -> int:
    """mix_seed (runner.cpp:175-180)."""
    x = (seed ^ (salt * 0x9E3779B97F4A7C15)) & _MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


def make_problem(c: RunConfig, seed: int):
    """make_problem (runner.cpp:182-204): (p, q), uniform marginals."""
    if c.generator == "uniform-ball":
        p = N.sample_uniform_ball(c.n, c.d, mix_seed(seed, 1))
        q = N.sample_uniform_ball(c.m or c.n, c.d, mix_seed(seed, 2))
    elif c.generator == "clustered":
        p, q, _ = N.sample_clustered(c.n, c.d, c.c, c.D, c.r, seed)
    else:
        p, q = N.read_points_file(c.path_p), N.read_points_file(c.path_q)
    return p, q


def lsh_bucket_count(c: RunConfig, n: int, m: int, neighbors: int) -> int:
    """lsh_bucket_count (runner.cpp:206-216): b^r = min(n, m) / beta."""
    if c.buckets_per_fn > 0:
        return c.buckets_per_fn
    target = min(n, m) / max(1, neighbors)
    per_fn = max(target, 2.0) ** (1.0 / c.rows_per_band)
    b = int(math.floor(per_fn + 0.5))  # llround: halves away from zero
    if _SCHEMES[c.lsh_scheme] == N.LSH_CROSS_POLYTOPE and b % 2:
        b += 1
    return max(b, 2)


# ---- plans on the device (densify_plan, sinkhorn.cpp:371-405) ---------------
def _dense_plan(op: N.KernelOperator, res: N.SinkhornResult):
    import torch
    dev = torch.device("cuda", op.ctx.device)
    n, m = op.n, op.m
    ls = torch.from_numpy(res.log_s).to(dev)
    lt = torch.from_numpy(res.log_t).to(dev)
    kind = op.info.kind
    if kind == N.KIND_DENSE:
        return torch.from_numpy(res.sparse_vals.reshape(n, m)).to(dev)
    out = torch.zeros((n, m), dtype=torch.float64, device=dev)
    if kind == N.KIND_SPARSE:
        rp, col, _ = op.export_csr(0)
        rows = torch.repeat_interleave(torch.arange(n, device=dev), torch.from_numpy(np.diff(rp).astype(np.int64)).to(dev))
        out[rows, torch.from_numpy(col.astype(np.int64)).to(dev)] = torch.from_numpy(res.sparse_vals).to(dev)
        return out
    pu = torch.exp(ls)[:, None] * torch.from_numpy(op.factor(0)).to(dev)
    pw = torch.from_numpy(op.factor(1)).to(dev) * torch.exp(lt)[None, :]
    out = pu @ pw
    if kind == N.KIND_LCN and op.nnz:
        rp, col, _ = op.export_csr(1)
        rows = torch.repeat_interleave(torch.arange(n, device=dev), torch.from_numpy(np.diff(rp).astype(np.int64)).to(dev))
        corr = torch.from_numpy(res.sp_vals - res.sp_nys_vals).to(dev)
        out.index_put_((rows, torch.from_numpy(col.astype(np.int64)).to(dev)), corr, accumulate=True)
    return out


def compare_plans(p_ref, p_app):
    """compare_plans (metrics.cpp:21-70): PCC and the IoU of the top-0.1%
    entries (ties by value desc, then linear index asc); None when a plan is
    constant (PccUndefinedError)."""
    import torch
    a, b = p_ref.reshape(-1), p_app.reshape(-1)
    xa, xb = a - a.mean(), b - b.mean()
    va, vb = float((xa * xa).sum()), float((xb * xb).sum())
    if va == 0.0 or vb == 0.0:
        return None, None
    pcc = float((xa * xb).sum()) / math.sqrt(va * vb)
    k = int(math.ceil(0.001 * a.numel()))
    ta = torch.sort(a, descending=True, stable=True).indices[:k]
    tb = torch.sort(b, descending=True, stable=True).indices[:k]
    inter = int(torch.isin(ta, tb).sum())
    return pcc, inter / (2 * k - inter)


@dataclasses.dataclass
class _SeedContext:
    p: np.ndarray
    q: np.ndarray
    ref: Optional[N.SinkhornResult] = None
    ref_plan: object = None


def _opts(c: RunConfig):
    return N.SinkhornOptions(tol=c.tol, max_iters=c.max_iters)


def run_one(ctx: N.Context, c: RunConfig, variant: str, seed: int, sc: _SeedContext) -> dict:
    """run_one (runner.cpp:230-330) on the GPU operators."""
    p, q = sc.p, sc.q
    n, m = p.shape[0], q.shape[0]
    budget = {"sparse": c.neighbors, "nystrom": c.landmarks, "lcn": c.neighbors + c.landmarks}.get(variant, 0)
    rec = {"variant": variant, "seed": seed, "n": n, "m": m, "lambda": c.lam, "budget": budget, "distance": 0.0,
           "converged": False, "iters": 0, "marginal-err": 0.0}
    cost = _COSTS[c.cost]
    pm, qm = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    try:
        t0 = time.perf_counter()
        if variant == "full":
            op = N.KernelOperator.dense(ctx, p, q, cost, c.lam)
        elif variant in ("sparse", "lcn"):
            cfg = N.LshConfig(c.bands, c.rows_per_band, lsh_bucket_count(c, n, m, c.neighbors), c.kmeans_iters,
                              mix_seed(seed, 3), _SCHEMES[c.lsh_scheme], c.branching)
            if variant == "sparse":
                op = N.KernelOperator.sparse_lsh(ctx, p, q, cost, c.lam, cfg)
            else:
                op = N.KernelOperator.lcn_lsh(ctx, p, q, cost, c.lam, cfg, max(1, c.landmarks),
                                              _LANDMARKS[c.landmark_method], mix_seed(seed, 4))
        elif variant == "nystrom":
            op = N.KernelOperator.lcn_buckets(ctx, p, q, cost, c.lam, None, None, max(1, c.landmarks),
                                              _LANDMARKS[c.landmark_method], mix_seed(seed, 4))
        else:
            raise N.InvalidArgument(f"unknown variant '{variant}'")
        if c.bp:  # runner.cpp:282-286: scalar deletion cost on both sides
            op.with_bp(np.full(n, c.deletion_cost), np.full(m, c.deletion_cost))
        ms_kernel = (time.perf_counter() - t0) * 1e3
        t1 = time.perf_counter()
        if c.heads > 1 and variant == "full":
            heads = N.multihead(ctx, p, q, cost, c.lam, c.heads, pm, qm, _opts(c))
            for h in heads:
                if h["error"]:
                    raise N.Error(f"head λ={h['lambda']:f}: {h['error']}")
            rec["head-distances"] = [h["distance"] for h in heads]
        res = N.sinkhorn(op, pm, qm, _opts(c))
        ms_ot = (time.perf_counter() - t1) * 1e3
        rec.update({"distance": res.distance, "converged": res.converged, "iters": res.iters,
                    "marginal-err": res.marginal_err_final})
        if sc.ref is not None and not c.bp:
            rec["rel-err-d"] = abs(res.distance - sc.ref.distance) / abs(sc.ref.distance)
            pcc, iou = compare_plans(sc.ref_plan, _dense_plan(op, res))
            if pcc is not None:
                rec["pcc"], rec["iou"] = pcc, iou
        if not c.strict_deterministic:
            rec["ms-kernel"], rec["ms-ot"] = ms_kernel, ms_ot
    except N.Error as e:
        rec["error"] = f"{e} [variant={variant} seed={seed}]"
    # key order of record_to_json
    order = ["variant", "seed", "n", "m", "lambda", "budget", "distance", "converged", "iters", "marginal-err",
             "rel-err-d", "pcc", "iou", "ms-kernel", "ms-ot", "error", "head-distances"]
    return {k: rec[k] for k in order if k in rec}


def run_all(c: RunConfig, ctx: Optional[N.Context] = None) -> list:
    """run_all (runner.cpp:344-418): per seed the problem and, when n m <=
    10^6 and no BP, the dense reference solve; then every (variant, seed)."""
    if not c.variants:
        raise N.InvalidArgument("run: no variants requested")
    ctx = ctx or N.Context(0)
    scs = []
    for seed in c.seeds:
        p, q = make_problem(c, seed)
        sc = _SeedContext(p, q)
        if p.shape[0] * q.shape[0] <= 1_000_000 and not c.bp:
            op = N.KernelOperator.dense(ctx, p, q, _COSTS[c.cost], c.lam)
            sc.ref = N.sinkhorn(op, np.full(p.shape[0], 1.0 / p.shape[0]), np.full(q.shape[0], 1.0 / q.shape[0]),
                                _opts(c))
            sc.ref_plan = _dense_plan(op, sc.ref)
        scs.append(sc)
    return [run_one(ctx, c, v, seed, sc) for v in c.variants for seed, sc in zip(c.seeds, scs)]


def _csv_num(v) -> str:
    return "" if v is None else format(v, ".10g")


CSV_HEADER = "variant,n,m,lambda,budget,rel_err_d,pcc,iou,iters,ms_kernel,ms_ot"  # metrics.cpp:327-330


def csv_row(r: dict) -> str:
    """sweep_csv_row (metrics.cpp:343-351), precision 10."""
    return ",".join([r["variant"], str(r["n"]), str(r["m"]), _csv_num(r["lambda"]), str(r["budget"]),
                     _csv_num(r.get("rel-err-d")), _csv_num(r.get("pcc")), _csv_num(r.get("iou")), str(r["iters"]),
                     _csv_num(r.get("ms-kernel")), _csv_num(r.get("ms-ot"))])


def write_outputs(c: RunConfig, records: list, json_path: str = "") -> int:
    """write_outputs (runner.cpp:420-445): CSV rows of the successful records
    (stdout or config.output), optional JSON {config, records}; exit code 2
    when any record failed."""
    out = open(c.output, "w") if c.output else sys.stdout
    try:
        out.write(CSV_HEADER + "\n")
        for r in records:
            if "error" not in r:
                out.write(csv_row(r) + "\n")
    finally:
        if c.output:
            out.close()
    if json_path:
        with open(json_path, "w") as f:
            f.write(json.dumps({"config": config_to_json(c), "records": records}, indent=2, ensure_ascii=False) + "\n")
    code = 0
    for r in records:
        if "error" in r:
            print(f"lcn: variant failed: {r['error']}", file=sys.stderr)
            code = 2
    return code


def main(argv=None) -> int:
    """`python -m paper_2107_06876_b200.runner CONFIG.json [RECORDS.json]`."""
    argv = sys.argv[1:] if argv is None else argv
    with open(argv[0]) as f:
        cfg = config_from_json(json.load(f))
    return write_outputs(cfg, run_all(cfg), argv[1] if len(argv) > 1 else "")


if __name__ == "__main__":
    sys.exit(main())
