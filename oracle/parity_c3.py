"""ORACLE TEST INFRASTRUCTURE: full-size parity of configs[3] against the
compiled reference (oracle/_ref/libref_lcn.so).

The headline workload (n = m = 10^6, d = 128, 2 x 4096 k-means LSH, l = 512,
100 iterations) is too large for the unit suite, so this script runs the
reference's own staged path on the host and compares it with a dump of the
GPU path (scripts/parity_c3_gpu.py, run on the B200 box). Stages:

  lsh        reference k-means LSH, one band per host thread:
             hash_kmeans(union, fn_seed(seed, band, 0)) (lsh.cpp:267-281)
             -> SCRATCH/ref_ids.npz                               (~1-2 h)
  landmarks  select_landmarks(l = 512, KMeans) (nystrom.cpp:28-48)
             -> SCRATCH/ref_landmarks.npy                         (~10 min)
  pipeline   from bucket ids (--ids: the GPU's, or the reference's own) and
             the reference landmarks: neighbor_pairs(BandBuckets...)
             (lsh.cpp:212-243) -> build_sparse -> build_factors (restated,
             Eigen absent) -> build_correction -> KernelOperator::lcn ->
             sinkhorn(tol 0, 100 iterations, want_plan false), each stage
             timed; then the per-row support digest, extract_plan entries of
             400 seeded rows, log s / log t -> SCRATCH/ref_pipeline.npz
  compare    GPU dump vs the reference outputs -> profiles/parity_c3_full.json

SCRATCH defaults to <repo>/scratch (git- and gpurun-ignored).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.bindings import RefLib  # noqa: E402
from paper_2107_06876_b200 import configs  # noqa: E402

SAMPLE_ROWS = 400
SAMPLE_SEED = 20261020


def mix64(x: np.ndarray) -> np.ndarray:
    """lsh.cpp:17-22 over uint64 arrays (the digest's column hash)."""
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def row_digest_np(row_ptr: np.ndarray, col: np.ndarray):
    """Same digest as ref_op_row_digest, from a host CSR (numpy)."""
    n = len(row_ptr) - 1
    cnt = np.diff(row_ptr.astype(np.int64)).astype(np.uint32)
    hs = np.zeros(n, np.uint64)
    hx = np.zeros(n, np.uint64)
    nz = cnt > 0
    starts = row_ptr[:-1].astype(np.int64)[nz]
    step = 1 << 26
    h = np.empty(len(col), np.uint64)
    for o in range(0, len(col), step):  # bounded temporaries
        h[o:o + step] = mix64(col[o:o + step])
    with np.errstate(over="ignore"):
        hs[nz] = np.add.reduceat(h, starts)
    hx[nz] = np.bitwise_xor.reduceat(h, starts)
    return cnt, hs, hx


def sample_rows(n: int) -> np.ndarray:
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.sort(rng.choice(n, SAMPLE_ROWS, replace=False)).astype(np.uint32)


def stage_lsh(args, pr, ref):
    all_pts = np.concatenate([pr.p, pr.q])
    ids = np.zeros((pr.bands, pr.n + pr.m), np.uint64)
    secs = [0.0] * pr.bands

    def band(b):
        t0 = time.perf_counter()
        ids[b] = ref.hash_kmeans_band(all_pts, pr.buckets, pr.kmeans_iters, pr.lsh_seed, b)
        secs[b] = time.perf_counter() - t0
        print(f"band {b}: {secs[b]:.1f} s", flush=True)

    th = [threading.Thread(target=band, args=(b,)) for b in range(pr.bands)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    np.savez_compressed(os.path.join(args.scratch, "ref_ids.npz"), ids=ids, n=pr.n, band_s=np.array(secs))


def stage_landmarks(args, pr, ref):
    t0 = time.perf_counter()
    lm = ref.select_landmarks(pr.p, pr.q, pr.landmarks, configs.LANDMARK_KMEANS, pr.landmark_seed)
    dt = time.perf_counter() - t0
    np.save(os.path.join(args.scratch, "ref_landmarks.npy"), lm)
    json.dump({"select_landmarks_s": dt}, open(os.path.join(args.scratch, "ref_landmarks.json"), "w"))
    print(f"landmarks: {dt:.1f} s", flush=True)


def stage_pipeline(args, pr, ref):
    ids = np.load(args.ids)["ids"].astype(np.uint64)
    lm = np.load(os.path.join(args.scratch, "ref_landmarks.npy"))
    ids_p, ids_q = np.ascontiguousarray(ids[:, :pr.n]), np.ascontiguousarray(ids[:, pr.n:])
    t0 = time.perf_counter()
    op, phases = ref.lcn_pipeline(pr.p, pr.q, pr.cost, pr.lam_eff, ids_p, ids_q, pr.buckets, lm)
    print("build:", phases, f"wall {time.perf_counter() - t0:.1f} s", flush=True)
    nnz = op.nnz
    cnt, hs, hx = ref.row_digest(op)
    pm, qm = pr.marginals()
    t1 = time.perf_counter()
    res = op.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters, check_support=False, want_plan=False)
    t_it = time.perf_counter() - t1
    print(f"sinkhorn {pr.iters} iterations: {t_it:.1f} s, distance {res.distance!r}", flush=True)
    rows = sample_rows(pr.n)
    pl = ref.plan_rows(op, res, rows, cnt)
    dl = res.distance_lcn()
    np.savez(os.path.join(args.scratch, "ref_pipeline.npz"), cnt=cnt, hs=hs, hx=hx, log_s=res.log_s,
             log_t=res.log_t, rows=rows, err=res.marginal_err, **{f"pl_{k}": v for k, v in pl.items()})
    meta = {"ids": os.path.basename(args.ids), "nnz": int(nnz), "distance": res.distance, "distance_lcn": dl,
            "mu": pr.mu, "iters": res.iters, "phases_s": phases, "iterations_s": t_it,
            "iter_per_s": pr.iters / t_it, "threads": int(os.environ.get("OMP_NUM_THREADS", "0")),
            "host_cores": os.cpu_count()}
    json.dump(meta, open(os.path.join(args.scratch, "ref_pipeline.json"), "w"), indent=1)
    print(json.dumps(meta), flush=True)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def stage_compare(args, pr, ref):
    sc = args.scratch
    g = np.load(args.gpu)
    gmeta = json.loads(str(g["meta"]))
    out = {"config": "configs[3] full: n=m=1e6, d=128, sqL2/mean, lambda=0.05, 2x4096 k-means LSH, l=512, "
                     "100 iterations, tol 0", "gpu": gmeta}
    ids_gpu = g["ids"].astype(np.uint64)
    if os.path.exists(os.path.join(sc, "ref_ids.npz")):
        rz = np.load(os.path.join(sc, "ref_ids.npz"))
        ids_ref = rz["ids"]
        out["bucket_ids"] = {"points": int(ids_ref.size), "mismatches": int((ids_ref != ids_gpu).sum()),
                             "bit_exact": bool(np.array_equal(ids_ref, ids_gpu)),
                             "reference_lsh_s_per_band": [float(x) for x in rz["band_s"]]}
    lm_ref = np.load(os.path.join(sc, "ref_landmarks.npy"))
    out["landmarks"] = {"bit_exact": bool(np.array_equal(lm_ref.view(np.uint64), g["landmarks"].view(np.uint64))),
                        "mismatched_values": int((lm_ref != g["landmarks"]).sum())}
    rp = np.load(os.path.join(sc, "ref_pipeline.npz"))
    rmeta = json.load(open(os.path.join(sc, "ref_pipeline.json")))
    out["reference"] = rmeta
    out["support"] = {"nnz_ref": rmeta["nnz"], "nnz_gpu": gmeta["nnz"],
                      "row_counts_equal": bool(np.array_equal(rp["cnt"], g["cnt"])),
                      "row_digests_equal": bool(np.array_equal(rp["hs"], g["hs"]) and np.array_equal(rp["hx"], g["hx"])),
                      "rows_differing": int(((rp["cnt"] != g["cnt"]) | (rp["hs"] != g["hs"]) | (rp["hx"] != g["hx"])).sum())}
    mu = pr.mu
    for tag in ("fp32", "fp64"):
        if f"{tag}_distance" not in gmeta:
            continue
        d_g, d_r = gmeta[f"{tag}_distance"], rmeta["distance"]
        blk = {"distance_gpu": d_g / mu, "distance_ref": d_r / mu, "distance_rel": float(rel(d_g, d_r)),
               "distance_lcn_rel": float(rel(gmeta[f"{tag}_distance_lcn"], rmeta["distance_lcn"]))}
        if f"{tag}_sp_vals" in g:
            same_cols = np.array_equal(g["pl_cols"], rp["pl_cols"])
            blk["sampled_rows"] = int(len(rp["rows"]))
            blk["sampled_entries"] = int(len(rp["pl_cols"]))
            blk["sampled_cols_equal"] = bool(same_cols)
            if same_cols:
                r_sp = rel(g[f"{tag}_sp_vals"], rp["pl_sp_vals"])
                r_ny = rel(g[f"{tag}_sp_nys_vals"], rp["pl_sp_nys_vals"])
                blk["sp_vals_max_rel"] = float(r_sp.max())
                blk["sp_vals_median_rel"] = float(np.median(r_sp))
                blk["sp_nys_vals_max_rel"] = float(r_ny.max())
                blk["log_sp_bit_exact"] = bool(np.array_equal(g["pl_log_sp"].view(np.uint64),
                                                              rp["pl_log_sp"].view(np.uint64)))
                blk["delta_max_abs"] = float(np.abs(g[f"{tag}_delta"] - rp["pl_delta"]).max())
        if f"{tag}_log_s" in g:
            # scalings are defined up to the gauge s -> a s, t -> t / a (sinkhorn.hpp:118-120):
            # compare the gauge-free sums log s_i + log t_j through the plan instead, and the
            # raw vectors after removing the mean shift
            ls_g, lt_g = g[f"{tag}_log_s"], g[f"{tag}_log_t"]
            shift = float(np.mean(ls_g - rp["log_s"]))
            blk["log_s_gauge_shift"] = shift
            blk["log_s_max_abs_after_gauge"] = float(np.abs(ls_g - shift - rp["log_s"]).max())
            blk["log_t_max_abs_after_gauge"] = float(np.abs(lt_g + shift - rp["log_t"]).max())
        out[tag] = blk
    bar = 1e-4
    ok = out.get("fp32", {})
    out["pass"] = {"support_bit_exact": out["support"]["row_digests_equal"] and rmeta["nnz"] == gmeta["nnz"],
                   "bucket_ids_bit_exact": out.get("bucket_ids", {}).get("bit_exact"),
                   "landmarks_bit_exact": out["landmarks"]["bit_exact"],
                   "distance_within_1e-4": ok.get("distance_rel", 1.0) <= bar,
                   "sp_vals_within_1e-4": ok.get("sp_vals_max_rel", 1.0) <= bar}
    path = args.out or os.path.join(ROOT, "profiles", "parity_c3_full.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out["pass"]), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("stage", choices=["lsh", "landmarks", "pipeline", "compare"])
    ap.add_argument("--scratch", default=os.path.join(ROOT, "scratch"))
    ap.add_argument("--ids", default=None, help="npz with ids (bands x (n+m)) for the pipeline stage")
    ap.add_argument("--gpu", default=None, help="GPU dump npz (scripts/parity_c3_gpu.py) for compare")
    ap.add_argument("--out", default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    os.makedirs(args.scratch, exist_ok=True)
    pr = configs.config3(args.scale)
    ref = RefLib()
    {"lsh": stage_lsh, "landmarks": stage_landmarks, "pipeline": stage_pipeline,
     "compare": stage_compare}[args.stage](args, pr, ref)


if __name__ == "__main__":
    main()
