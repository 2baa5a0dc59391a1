"""GPU half of the full-size configs[3] parity check (test infrastructure;
oracle/parity_c3.py holds the reference half and the comparison).

Runs on the B200 box through the product's host-buffer C-ABI entry
(lcn_op_lcn_lsh: fp64 host points -> k-means LSH, landmarks, factors,
correction, all on the device) and lcn_sinkhorn (tol 0, 100 iterations, plan
extracted), in both storage modes, and writes what the reference side needs:
bucket ids of both bands, the landmarks, the per-row support digest, the
scalings and the plan entries of the same 400 seeded rows.

usage: python tests/parity_c3_gpu.py OUT.npz [scale]
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2107_06876_b200 as lcn  # noqa: E402
from paper_2107_06876_b200 import configs  # noqa: E402
from oracle.parity_c3 import row_digest_np, sample_rows  # noqa: E402  (checker only)


def main():
    out = sys.argv[1]
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    pr = configs.config3(scale)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    pm, qm = pr.marginals()
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, check_support=False, want_plan=True)
    rows = sample_rows(pr.n)
    dump, meta = {"rows": rows}, {"n": pr.n, "scale": scale}

    ctx = lcn.Context(0)
    t0 = time.perf_counter()
    ids = lcn.lsh_kmeans_buckets(ctx, pr.p, pr.q, cfg)
    meta["lsh_s"] = time.perf_counter() - t0
    dump["ids"] = ids.astype(np.uint16 if pr.buckets <= 65536 else np.uint64)

    for tag, store64 in (("fp32", False), ("fp64", True)):
        c = lcn.Context(0, store_fp64=store64) if store64 else ctx
        t0 = time.perf_counter()
        op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks,
                                        lcn.LANDMARK_KMEANS, pr.landmark_seed)
        meta[f"{tag}_build_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = lcn.sinkhorn(op, pm, qm, opts)
        meta[f"{tag}_solve_s"] = time.perf_counter() - t0
        meta[f"{tag}_distance"] = res.distance
        meta[f"{tag}_distance_lcn"] = lcn.distance_lcn(res, op)
        meta[f"{tag}_iters"] = res.iters
        rp, col, log_sp = op.export_csr(2)
        if tag == "fp32":
            meta["nnz"] = int(op.nnz)
            meta["stored"] = int(op.stored)
            dump["landmarks"] = op.factor(2)
            dump["cnt"], dump["hs"], dump["hx"] = row_digest_np(rp, col)
            dump["fp32_log_s"], dump["fp32_log_t"] = res.log_s, res.log_t
        sel = np.concatenate([np.arange(rp[i], rp[i + 1], dtype=np.int64) for i in rows])
        if tag == "fp32":
            dump["pl_cols"] = col[sel]
            dump["pl_log_sp"] = log_sp[sel]
        del col, log_sp
        dump[f"{tag}_delta"] = op.export_csr(1)[2][sel]
        dump[f"{tag}_sp_vals"] = res.sp_vals[sel]
        dump[f"{tag}_sp_nys_vals"] = res.sp_nys_vals[sel]
        print(tag, json.dumps({k: v for k, v in meta.items() if k.startswith(tag)}), flush=True)
        del res, op
        if store64:
            c.close()
    dump["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(out, **dump)
    print("saved", out, json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
