"""GPU parity: the CUDA path (C-ABI) against the reference compiled from its own
sources (oracle/_ref) on the same seeded inputs.

Bar (BASELINE.json north_star): bucket ids and sparse support bit-exact;
Sinkhorn distance and plan entries within 1e-4 relative (fp32 storage) —
1e-9 with fp64 storage.
"""
import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

pytestmark = pytest.mark.gpu

REL_FP32 = 1e-4
REL_FP64 = 1e-9


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def rng_points(seed, n, d, comps=5, spread=3.0):
    r = np.random.default_rng(seed)
    means = r.standard_normal((comps, d)) * spread
    return (means[r.integers(0, comps, n)] + r.standard_normal((n, d))).astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("n,d,k,seed", [(40, 3, 4, 1), (500, 8, 16, 7), (4000, 32, 16, 3), (3000, 300, 37, 11),
                                        (64, 2, 60, 5)])
def test_lloyd_bit_exact(ctx, ref, n, d, k, seed):
    x = rng_points(seed, n, d)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, k, 10, seed)
    c_ref, a_ref = ref.lloyd(x, k, 10, seed)
    assert np.array_equal(a_gpu, a_ref)
    assert np.array_equal(c_gpu.view(np.uint64), c_ref.view(np.uint64))


@pytest.mark.parametrize("n,d,k,seed", [(50, 2, 50, 3), (1000, 16, 64, 9), (20000, 8, 33, 4)])
def test_kmeans_pp_bit_exact(ctx, ref, n, d, k, seed):
    x = rng_points(seed, n, d)
    assert np.array_equal(lcn.kmeans_pp_indices(ctx, x, k, seed=seed), ref.kmeans_pp(x, k, seed))


@pytest.mark.parametrize("kind", ["mixture", "outliers", "duplicates"])
def test_kmeans_pp_large_walk(ctx, ref, kind):
    # ~700 fold chunks: clean runs, binade-crossing segments, huge elements
    # (outliers far away) and runs of zeros (duplicated points)
    n, d, k = 1_400_000, 3, 24
    x = rng_points(77, n, d, comps=12)
    if kind == "outliers":
        r = np.random.default_rng(78)
        x[r.choice(n, 50, replace=False)] *= 1e5
    elif kind == "duplicates":
        x[: n // 2] = x[0]
    assert np.array_equal(lcn.kmeans_pp_indices(ctx, x, k, seed=9), ref.kmeans_pp(x, k, 9))


@pytest.mark.parametrize("mode", [{}, {"LCN_PP_EXACT_WALK": "1"}, {"LCN_PP_CERT_SLACK": "20000"},
                                  {"LCN_PP_CERT_SLACK": "1e9"}])
def test_kmeans_pp_certified_pick(ctx, ref, monkeypatch, mode):
    # the certified pick (pp_pick_kernel) and the exact fold + walk give
    # the same indices: default (almost every step certified), exact walk
    # only, a widened certificate (about half the steps fall back, so the two
    # paths alternate) and one so wide that every step falls back
    for key, val in mode.items():
        monkeypatch.setenv(key, val)
    n, d, k = 200_000, 8, 96
    x = rng_points(91, n, d, comps=20)
    assert np.array_equal(lcn.kmeans_pp_indices(ctx, x, k, seed=13), ref.kmeans_pp(x, k, 13))


def test_kmeans_pp_duplicates_total_zero(ctx, ref):
    # all points coincide: total <= 0 branch takes the first unused index (kmeans.cpp:42-47)
    x = np.zeros((12, 3))
    assert np.array_equal(lcn.kmeans_pp_indices(ctx, x, 6, seed=5), ref.kmeans_pp(x, 6, 5))


def test_assign_ties_lowest_index(ctx, ref):
    x = np.array([[0.0], [1.0], [2.0]])
    ctr = np.array([[1.0], [1.0], [0.0], [0.0]])
    assert np.array_equal(lcn.assign_nearest(ctx, x, ctr), ref.assign_nearest(x, ctr))


@pytest.mark.parametrize("n,d,k,seed,dup", [(40000, 128, 128, 21, False), (50000, 37, 96, 22, False),
                                            (40000, 64, 128, 23, True)])
def test_assign_filter_bit_exact(ctx, ref, n, d, k, seed, dup):
    # N k >= 2^22 with fp32 points: the fp32 filter + exact fallback path.
    # dup: centroids 64.. repeat 0.. -> exact ties, lowest index wins
    x = rng_points(seed, n, d)
    r = np.random.default_rng(seed)
    ctr = x[r.choice(n, k, replace=False)] + r.standard_normal((k, d)) * 0.3  # fp64, not fp32-exact
    if dup:
        ctr[k // 2:] = ctr[:k // 2]
    assert np.array_equal(lcn.assign_nearest(ctx, x, ctr), ref.assign_nearest(x, ctr))


def test_tc_work_counter(ctx, ref):
    # lcn_ctx_tc_work (bench.py's distance roofline): a full assignment
    # evaluates every point against every 128-centroid tile; Lloyd with its
    # bounds and tile skipping evaluates fewer than iters + 1 full ones
    n, d, k = 40000, 128, 256
    x = rng_points(31, n, d)
    r = np.random.default_rng(31)
    ctr = x[r.choice(n, k, replace=False)] + r.standard_normal((k, d)) * 0.3
    ctx.tc_work(reset=True)
    assert np.array_equal(lcn.assign_nearest(ctx, x, ctr), ref.assign_nearest(x, ctr))
    assert ctx.tc_work(reset=True) == n * (k // 128)
    n, k = 120000, 1024
    x = rng_points(32, n, d, comps=64)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, k, 10, 32)
    work = ctx.tc_work()
    assert 0 < work < 11 * n * (k // 128)
    assert ctx.tc_work(reset=True) == work and ctx.tc_work() == 0


@pytest.mark.parametrize("dup", [False, True])
def test_assign_gemm_filter_bit_exact(ctx, ref, dup):
    # d > 128 with N k >= 2^22: the fp32 GEMM + top-2 filter (configs[1]'s
    # d = 300) and its exact fallback; dup: exact ties, lowest index wins
    n, d, k = 40000, 300, 128
    x = rng_points(25, n, d, comps=30)
    r = np.random.default_rng(25)
    ctr = x[r.choice(n, k, replace=False)] + r.standard_normal((k, d)) * 0.3
    if dup:
        ctr[k // 2:] = ctr[:k // 2]
    assert np.array_equal(lcn.assign_nearest(ctx, x, ctr), ref.assign_nearest(x, ctr))


def test_lloyd_gemm_filter_bit_exact(ctx, ref):
    x = rng_points(27, 40000, 300, comps=50)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, 128, 10, 27)
    c_ref, a_ref = ref.lloyd(x, 128, 10, 27)
    assert np.array_equal(a_gpu, a_ref)
    assert np.array_equal(c_gpu.view(np.uint64), c_ref.view(np.uint64))


def test_lloyd_filter_bit_exact(ctx, ref):
    x = rng_points(31, 30000, 64, comps=40)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, 160, 10, 31)
    c_ref, a_ref = ref.lloyd(x, 160, 10, 31)
    assert np.array_equal(a_gpu, a_ref)
    assert np.array_equal(c_gpu.view(np.uint64), c_ref.view(np.uint64))


def test_lloyd_bounds_bit_exact(ctx, ref):
    # Lloyd with certified distance bounds (only bound-failing points are
    # re-assigned) against the reference: N k >= 2^22 with fp32 points
    x = rng_points(41, 60000, 32, comps=60)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, 256, 10, 41)
    c_ref, a_ref = ref.lloyd(x, 256, 10, 41)
    assert np.array_equal(a_gpu, a_ref)
    assert np.array_equal(c_gpu.view(np.uint64), c_ref.view(np.uint64))


def test_lloyd_bounds_match_full_reassignment(ctx, monkeypatch):
    # configs[3]-like mixture at 300k points, 1024 centroids: the bounded
    # iterations give the same assignment and centroid bits as re-assigning
    # every point every iteration
    r = np.random.default_rng(43)
    means = r.standard_normal((300, 128))
    x = (means[r.integers(0, 300, 300_000)] + 0.5 * r.standard_normal((300_000, 128))).astype(np.float32)
    x = x.astype(np.float64)
    c1, a1 = lcn.lloyd(ctx, x, 1024, 10, 43)
    monkeypatch.setenv("LCN_LLOYD_BOUNDS", "0")
    c0, a0 = lcn.lloyd(ctx, x, 1024, 10, 43)
    assert np.array_equal(a1, a0)
    assert np.array_equal(c1.view(np.uint64), c0.view(np.uint64))


def test_lsh_buckets_config0(ctx, ref):
    pr = configs.config0()
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    ids = lcn.lsh_kmeans_buckets(ctx, pr.p, pr.q, cfg)
    ids_ref = ref.lsh_buckets(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    assert np.array_equal(ids, ids_ref)


def _sparse_pair(ctx, ref, pr):
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    op = lcn.KernelOperator.sparse_lsh(ctx, pr.p, pr.q, pr.cost, pr.lam_eff, cfg)
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_sparse(pr.p, pr.q, pr.cost, pr.lam_eff, pairs)
    return op, rop


@pytest.mark.parametrize("mode", ["fp32_tc", "fp32_exact", "fp64"])
def test_sparse_config0_end_to_end(ref, mode):
    c = lcn.Context(0, store_fp64=mode == "fp64", exact_build=mode == "fp32_exact")
    fp64 = mode == "fp64"
    pr = configs.config0()
    op, rop = _sparse_pair(c, ref, pr)
    rp, col, lk = op.export_csr(0)
    rrp, rcol, rlk = rop.csr(0)
    assert np.array_equal(rp, rrp) and np.array_equal(col, rcol)          # support bit-exact
    if mode == "fp32_tc":  # tensor-core distance blocks: K within 1e-4 (|d log K| <= 1e-4)
        assert np.max(np.abs(lk - rlk)) <= 1e-4
    else:  # exact fp64 tiles: log K bit-exact
        assert np.array_equal(lk.view(np.uint64), rlk.view(np.uint64))
    pm, qm = pr.marginals()
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    tol = REL_FP64 if fp64 else REL_FP32
    assert res.iters == rres.iters == pr.iters
    assert rel(res.distance, rres.distance) <= tol
    assert rel(res.sparse_vals, rres.sparse_vals) <= tol
    assert len(res.warnings) == rres.n_warnings
    assert rel(res.marginal_err, rres.marginal_err) <= 1e-3


def test_sparse_empty_row_is_stabilization_error(ctx, ref):
    # source 1 alone in its bucket: its row is empty (sinkhorn.cpp:16-21; test_sinkhorn.cpp:241-248)
    p = rng_points(1, 3, 2)
    q = rng_points(2, 3, 2)
    ids_p = np.array([[0, 5, 1]], np.uint64)
    ids_q = np.array([[0, 1, 1]], np.uint64)
    op = lcn.KernelOperator.sparse_buckets(ctx, p, q, lcn.EUCLIDEAN, 0.5, ids_p, ids_q)
    with pytest.raises(lcn.StabilizationError, match="sparse"):
        lcn.sinkhorn(op, np.full(3, 1 / 3), np.full(3, 1 / 3), lcn.SinkhornOptions(check_support=False))


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("scale,which", [(0.05, 1), (0.002, 3)])
def test_lcn_small_configs(ref, scale, which, exact):
    pr = configs.config1(scale) if which == 1 else configs.config3(scale)
    c = lcn.Context(0, store_fp64=False, exact_build=exact)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    rp, col, dl = op.export_csr(1)
    rrp, rcol, rdl = rop.csr(1)
    assert np.array_equal(rp, rrp) and np.array_equal(col, rcol)
    scale_k = max(np.max(np.abs(rdl)), 1e-300)
    if exact:  # exact fp64 tiles
        assert np.max(np.abs(dl - rdl)) <= 1e-8 * max(scale_k, 1.0)
    else:  # 3xTF32 distance blocks and SDDMM (K^sp <= 1): absolute 1e-4
        assert np.max(np.abs(dl - rdl)) <= 1e-4
    pm, qm = pr.marginals()
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    assert rel(res.distance, rres.distance) <= REL_FP32
    assert rel(res.sp_vals, rres.sp_vals) <= REL_FP32
    assert rel(lcn.distance_lcn(res, op), rres.distance_lcn()) <= REL_FP32


@pytest.mark.parametrize("fp64", [False, True])
def test_build_schedules_agree(monkeypatch, fp64):
    # the build's scheduling choices change when work runs, never what it
    # computes: landmarks + factors on an early job (default) or after the
    # LSH with the landmarks seeded in the bands' batched chain; the device
    # pool mapped up front or grown on demand -> bit-identical operators
    pr = configs.config3(0.01)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    pm, qm = pr.marginals()
    out = []
    for env in ({}, {"LCN_EARLY_FACTORS": "0", "LCN_POOL_RESERVE_GB": "8"}):
        for k in ("LCN_EARLY_FACTORS", "LCN_POOL_RESERVE_GB"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        c = lcn.Context(0, store_fp64=fp64)
        op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                        pr.landmark_seed)
        res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=20))
        out.append((op.factor(1), op.factor(2), op.export_csr(1), res.distance))
    (w0, l0, (rp0, c0, d0), x0), (w1, l1, (rp1, c1, d1), x1) = out
    assert np.array_equal(l0.view(np.uint64), l1.view(np.uint64))
    assert np.array_equal(w0.view(np.uint64), w1.view(np.uint64))
    assert np.array_equal(rp0, rp1) and np.array_equal(c0, c1)
    assert np.array_equal(d0.view(np.uint64), d1.view(np.uint64))
    assert x0 == x1


_LARGE_REF = {}


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("scale,which", [(1.0, 1), (0.1, 3)])
def test_lcn_large_configs(ref, scale, which, fp64):
    """Full configs[1] (n = m = 2e4, d = 300, 2 x 128 buckets, l = 200) and
    configs[3] at scale 0.1 (n = m = 1e5, 2 x 410 buckets, l = 512) against the
    compiled reference end to end (its own k-means LSH, landmarks, factors,
    correction, solve): support bit-exact, distance / distance_lcn and the plan
    entries on the support within the storage mode's bar. Full configs[3]:
    profiles/parity_c3_full.json."""
    pr = configs.config1(scale) if which == 1 else configs.config3(scale)
    c = lcn.Context(0, store_fp64=fp64)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    pm, qm = pr.marginals()
    key = (scale, which)
    if key not in _LARGE_REF:  # the reference side once per config (minutes of host time)
        pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
        rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
        del pairs
        rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters, check_support=False)
        _LARGE_REF[key] = dict(csr=rop.csr(1), iters=rres.iters, distance=rres.distance, sp_vals=rres.sp_vals,
                               distance_lcn=rres.distance_lcn())
        del rres, rop
    R = _LARGE_REF[key]
    rp, col, dl = op.export_csr(1)
    rrp, rcol, rdl = R["csr"]
    assert np.array_equal(rp, rrp) and np.array_equal(col, rcol)
    # configs[1]'s target is a rotated copy: the union's k-means never puts a
    # source and a target in one bucket, so its support is empty on both sides
    # and the LCN operator is its Nystrom part
    if len(dl):
        assert np.max(np.abs(dl - rdl)) <= (1e-8 if fp64 else 1e-4)
    del rp, col, dl
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, check_support=False))
    tol = REL_FP64 if fp64 else REL_FP32
    assert res.iters == R["iters"] == pr.iters
    assert rel(res.distance, R["distance"]) <= tol
    assert rel(res.sp_vals, R["sp_vals"]) <= tol
    assert rel(lcn.distance_lcn(res, op), R["distance_lcn"]) <= tol


@pytest.mark.parametrize("fp64", [False, True])
def test_lcn_wide_and_split_buckets(ref, fp64):
    """Two buckets of ~2000 x 2000: the band kernels cut them into <= 1024
    column tiles and several row pieces, so both split-output combines (row
    sums over column tiles, column sums over row pieces) run."""
    import dataclasses
    pr = dataclasses.replace(configs.config3(0.004), bands=1, buckets=2, landmarks=32, iters=30)
    c = lcn.Context(0, store_fp64=fp64)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    ids = lcn.lsh_kmeans_buckets(c, pr.p, pr.q, cfg)
    sizes = np.bincount(ids[0, pr.n:].astype(np.int64))
    assert sizes.max() > 1024
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    pm, qm = pr.marginals()
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    tol = REL_FP64 if fp64 else REL_FP32
    assert rel(res.distance, rres.distance) <= tol
    assert rel(res.sp_vals, rres.sp_vals) <= tol
    # repeat: split combines are order-fixed, results bit-identical run to run
    res2 = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
    assert res2.distance == res.distance
    assert np.array_equal(res2.sp_vals, res.sp_vals)


@pytest.mark.parametrize("n,m", [(5000, 3000), (8000, 2000), (6000, 1500)])
def test_lcn_one_dominant_bucket(ref, n, m):
    """One bucket holding every point (buckets = 1): the band planner must
    lengthen the stream pieces instead of exceeding the 8-bit piece index
    (these shapes threw 'more than 255 pieces')."""
    r = np.random.default_rng(n + m)
    p = r.standard_normal((n, 6)).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((m, 6)) * 0.9).astype(np.float32).astype(np.float64)
    p[:3] += 40.0  # a far clump: the second of the two buckets (the LSH needs >= 2)
    q[:3] += 40.0
    c = lcn.Context(0)
    cfg = lcn.LshConfig(1, 1, 2, 10, 5)
    op = lcn.KernelOperator.lcn_lsh(c, p, q, lcn.SQEUCLIDEAN, 2.0, cfg, 16, lcn.LANDMARK_KMEANS, 3)
    assert op.nnz >= (n - 3) * (m - 3)
    pairs = ref.lsh_pairs(p, q, 1, 2, 10, 5)
    rop = ref.op_lcn(p, q, lcn.SQEUCLIDEAN, 2.0, pairs, 16, 0, 3)
    pm, qm = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=20, want_plan=False))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=20, want_plan=False)
    assert rel(res.distance, rres.distance) <= REL_FP32


@pytest.mark.parametrize("fp64", [False, True])
def test_sharded_solve_single_rank(ref, fp64):
    """The bucket-sharded solve (§8(e)) through a real 1-rank NCCL
    communicator: the shard build and every exchange of the sharded loop run
    (ncclAllGather of the per-half-iteration record and of the result
    slices); the result matches the unsharded solve and the reference."""
    pr = configs.config3(0.002)
    pm, qm = pr.marginals()
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    c = lcn.Context(0, store_fp64=fp64)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False)
    base = lcn.sinkhorn(op, pm, qm, opts)
    cs = lcn.Context(0, store_fp64=fp64)
    cs.set_comm(1, 0, lcn.nccl_unique_id())
    sop = lcn.KernelOperator.lcn_lsh(cs, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                     pr.landmark_seed)
    res = lcn.sinkhorn(sop, pm, qm, opts)
    tol = 1e-12 if fp64 else 1e-9
    assert sop.nnz == op.nnz
    assert rel(res.distance, base.distance) <= tol
    assert np.max(np.abs(res.log_s - base.log_s)) <= 1e-9
    assert np.max(np.abs(res.log_t - base.log_t)) <= 1e-9
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    assert rel(res.distance, rres.distance) <= (REL_FP64 if fp64 else REL_FP32)
    with pytest.raises(lcn.InvalidArgument, match="sharded"):
        sop.log_matvec(np.zeros(pr.m))


@pytest.mark.parametrize("fp64,cost,lam,n,m", [(False, lcn.EUCLIDEAN, 0.05, 310, 260),
                                               (True, lcn.EUCLIDEAN, 0.05, 310, 260),
                                               (False, lcn.COSINE_DERIVED, 0.1, 310, 260),
                                               (False, lcn.NEGATIVE_DOT, 0.2, 310, 260),
                                               (False, lcn.EUCLIDEAN, 0.05, 1200, 2052),
                                               (False, lcn.EUCLIDEAN, 0.05, 5000, 5000),
                                               (True, lcn.EUCLIDEAN, 0.05, 5000, 5000)])
def test_dense_anchor(ref, fp64, cost, lam, n, m):
    """configs[2]-shaped dense operator (H19): log K bit-exact, distance and the
    dense plan against the reference's dense solve. Row lengths divisible by 4
    take the 16-byte streaming kernel (dense_lse4_kernel), others the scalar one."""
    r = np.random.default_rng(5)
    p = r.standard_normal((n, 12)).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((m, 12)) * 0.8 + 0.1).astype(np.float32).astype(np.float64)
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    c = lcn.Context(0, store_fp64=fp64)
    op = lcn.KernelOperator.dense(c, p, q, cost, lam)
    rop = ref.op_dense(p, q, cost, lam)
    lk, rlk = op.export_dense(), rop.dense_logk()
    assert np.array_equal(lk.view(np.uint64), rlk.view(np.uint64))   # bit-exact log K
    pm, qm = np.full(n, 1 / n), np.full(m, 1 / m)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=50))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=50)
    tol = REL_FP64 if fp64 else REL_FP32
    assert res.iters == rres.iters == 50
    assert rel(res.distance, rres.distance) <= tol
    assert rel(res.sparse_vals, rres.dense_plan) <= (1e-8 if fp64 else 1e-3)
    # the trace converges to the storage-precision floor: fp32 storage forms the
    # exponents and row sums in fp32 (~1e-6 relative), fp64 storage in fp64
    assert np.allclose(res.marginal_err, rres.marginal_err, rtol=1e-3, atol=1e-12 if fp64 else 2e-6)


@pytest.mark.parametrize("cost,lam,n,m,d", [(lcn.EUCLIDEAN, 0.05, 310, 260, 12),
                                             (lcn.EUCLIDEAN, 0.2, 1000, 777, 40),
                                             (lcn.NEGATIVE_DOT, 0.2, 300, 500, 300),
                                             (lcn.EUCLIDEAN, 0.05, 5000, 5000, 300)])
def test_dense_recompute(ref, cost, lam, n, m, d):
    """configs[2]'s dense operator with exp(-C/lambda) recomputed every
    half-iteration as a tcgen05 3xTF32 GEMM fused with the log-sum-exp
    (LCN_DENSE_RECOMPUTE, dense_tc.cu; no n x m storage) against the
    reference's dense solve: distance and the dense plan."""
    r = np.random.default_rng(7)
    p = r.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((m, d)) * 0.8 + 0.1).astype(np.float32).astype(np.float64)
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    c = lcn.Context(0, dense_recompute=True)
    op = lcn.KernelOperator.dense(c, p, q, cost, lam)
    rop = ref.op_dense(p, q, cost, lam)
    pm, qm = np.full(n, 1 / n), np.full(m, 1 / m)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=50))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=50)
    assert res.iters == rres.iters == 50
    assert rel(res.distance, rres.distance) <= REL_FP32
    if n * m <= 1e6:
        assert rel(res.sparse_vals, rres.dense_plan) <= 1e-3
        assert np.array_equal(op.export_dense().view(np.uint64), rop.dense_logk().view(np.uint64))


def test_dense_config2_full(ref):
    """configs[2] at full size (configs[1]'s points: n = m = 20000, d = 300,
    L2, lambda = 0.05, 50 iterations): the stored fp32 operator and the
    tcgen05 recompute against the reference's dense solve."""
    pr = configs.config1(1.0)
    pm, qm = pr.marginals()
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters, want_plan=False, check_support=False)
    rop = ref.op_dense(pr.p, pr.q, pr.cost, pr.lam_eff)
    want = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters, check_support=False, want_plan=False).distance
    del rop
    for recompute in (False, True):
        c = lcn.Context(0, dense_recompute=recompute)
        op = lcn.KernelOperator.dense(c, pr.p, pr.q, pr.cost, pr.lam_eff)
        got = lcn.sinkhorn(op, pm, qm, opts).distance
        assert rel(got, want) <= REL_FP32, (recompute, got, want)
        del op


@pytest.mark.parametrize("fp64", [False, True])
def test_multihead(ref, fp64):
    """multihead_lambdas + multihead (H20): lambda schedule, per-head distance,
    iterations and convergence against the reference."""
    r = np.random.default_rng(9)
    p = r.standard_normal((150, 6)).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((140, 6)) + 0.3).astype(np.float32).astype(np.float64)
    pm, qm = np.full(150, 1 / 150), np.full(140, 1 / 140)
    heads = 6
    c = lcn.Context(0, store_fp64=fp64)
    # tol well above the fp32-storage error floor: the stopping iteration is then
    # not decided by round-off
    out = lcn.multihead(c, p, q, lcn.EUCLIDEAN, 0.5, heads, pm, qm, lcn.SinkhornOptions(tol=1e-5, max_iters=300))
    lam, dist, iters, conv, err = ref.multihead(p, q, lcn.EUCLIDEAN, 0.5, heads, pm, qm, tol=1e-5, max_iters=300)
    assert [o["lambda"] for o in out] == list(lam)                       # same schedule bits
    for k in range(heads):
        assert out[k]["status"] == 0 and err[k] == 0
        assert rel(out[k]["distance"], dist[k]) <= (REL_FP64 if fp64 else REL_FP32)
        assert out[k]["converged"] == bool(conv[k])
        assert abs(out[k]["iters"] - iters[k]) <= (0 if fp64 else 2)
    with pytest.raises(lcn.InvalidArgument, match="heads"):
        lcn.multihead(c, p, q, lcn.EUCLIDEAN, 0.5, 0, pm, qm)


def test_grad_cost(ref):
    """grad_cost (§8(f) 1): LCN d/dU, d/dW, d/dlog K^sp(_Nys); sparse and dense
    d/dC; against the reference's Gradients."""
    pr = configs.config3(0.002)
    pm, qm = pr.marginals()
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    c = lcn.Context(0, store_fp64=True)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=30))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=30)
    for which in (1, 2, 3, 4):
        g, stale = lcn.grad_cost(res, op, which)
        rg, rstale = rres.grad_cost(which)
        assert stale == rstale == True  # tol = 0: never converged
        assert g.shape == rg.shape
        assert np.max(np.abs(g - rg)) <= 1e-7 * max(np.max(np.abs(rg)), 1e-300)
    # dense: d/dC is the plan
    r = np.random.default_rng(3)
    p = r.standard_normal((90, 5))
    q = r.standard_normal((80, 5))
    dop = lcn.KernelOperator.dense(c, p, q, lcn.EUCLIDEAN, 0.5)
    drop = ref.op_dense(p, q, lcn.EUCLIDEAN, 0.5)
    dres = lcn.sinkhorn(dop, np.full(90, 1 / 90), np.full(80, 1 / 80), lcn.SinkhornOptions(tol=1e-9, max_iters=500))
    drres = drop.sinkhorn(np.full(90, 1 / 90), np.full(80, 1 / 80), tol=1e-9, max_iters=500)
    g, stale = lcn.grad_cost(dres, dop, 0)
    rg, rstale = drres.grad_cost(0)
    assert not stale and not rstale
    assert rel(g, rg) <= 1e-8
    with pytest.raises(lcn.InvalidArgument):
        lcn.grad_cost(dres, dop, 1)


@pytest.mark.parametrize("layout", [{"LCN_PANEL_W": "1", "LCN_PANEL_A": "0"}, {},
                                    {"LCN_PANEL_W": "1000000"}, {"LCN_PANELS": "0"}, {"LCN_BAND_STATIC": "1"}])
@pytest.mark.parametrize("shape", ["c3", "three_bands", "wide"])
def test_lcn_panel_layouts(ref, monkeypatch, layout, shape):
    """The band streams of later bands skip the pairs band 0 already holds
    (gapped panels, BandPanel in op.cuh). Every panel policy — each band-0
    group its own panel, the default thresholds, all plain panels, the block
    layout — must give the reference's distance and support plan; `wide`
    forces gapped panels taller than one stream piece (split combines)."""
    import dataclasses
    for k, v in layout.items():
        monkeypatch.setenv(k, v)
    if shape == "c3":
        pr = configs.config3(0.02)
    elif shape == "three_bands":
        pr = dataclasses.replace(configs.config3(0.01), bands=3)
    else:
        pr = dataclasses.replace(configs.config3(0.004), bands=2, buckets=3, landmarks=32, iters=30)
    c = lcn.Context(0, store_fp64=False)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    pairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    if layout.get("LCN_PANELS") == "0" or layout.get("LCN_PANEL_W") == "1000000":
        assert op.streamed == op.stored
    else:
        assert op.nnz <= op.streamed < op.stored
    pm, qm = pr.marginals()
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    assert rel(res.distance, rres.distance) <= REL_FP32
    assert rel(res.sp_vals, rres.sp_vals) <= REL_FP32
    # log_matvec goes through the same band streams (both orientations)
    # (log domain: absolute 1e-4 = relative 1e-4 of K t; entries near log 1 = 0)
    for mine, theirs in [(op.log_matvec(rres.log_t), rop.log_matvec(rres.log_t)),
                         (op.log_matvec_t(rres.log_s), rop.log_matvec(rres.log_s, transposed=True))]:
        assert np.max(np.abs(mine - theirs) / np.maximum(np.abs(theirs), 1.0)) <= REL_FP32


def test_lcn_bands_without_two_sided_buckets(ref):
    """Sources and targets in separate far clusters: every LSH bucket of both
    bands is one-sided, so no band has work (empty support) and the LCN
    operator reduces to its Nystrom part — as in the reference."""
    r = np.random.default_rng(21)
    p = (r.standard_normal((300, 6)) * 0.3 + 4.0).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((280, 6)) * 0.3 - 4.0).astype(np.float32).astype(np.float64)
    c = lcn.Context(0, store_fp64=False)
    cfg = lcn.LshConfig(2, 1, 2, 10, 7)
    op = lcn.KernelOperator.lcn_lsh(c, p, q, lcn.EUCLIDEAN, 2.0, cfg, 12, lcn.LANDMARK_KMEANS, 3)
    pairs = ref.lsh_pairs(p, q, 2, 2, 10, 7)
    rop = ref.op_lcn(p, q, lcn.EUCLIDEAN, 2.0, pairs, 12, 0, 3)
    assert op.nnz == 0
    pm, qm = np.full(300, 1 / 300), np.full(280, 1 / 280)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=30))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=30)
    assert rel(res.distance, rres.distance) <= REL_FP32


def test_band_claim_order_does_not_change_results(monkeypatch):
    """Dynamic item claims (default) and static per-CTA ranges give bit-identical
    iterations: unsplit outputs are plain stores and split outputs are
    combined in piece order, whatever CTA processed them."""
    import dataclasses
    pr = dataclasses.replace(configs.config3(0.004), bands=2, buckets=3, landmarks=32, iters=30)
    out = []
    for static in (False, True):
        if static:
            monkeypatch.setenv("LCN_BAND_STATIC", "1")
        c = lcn.Context(0, store_fp64=False)
        cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
        op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                        pr.landmark_seed)
        pm, qm = pr.marginals()
        res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=pr.iters))
        out.append((res.distance, res.log_s.copy()))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1].view(np.uint64), out[1][1].view(np.uint64))


@pytest.mark.parametrize("exit_", ["1", "0"])
def test_lloyd_fixed_point_exit(ctx, ref, monkeypatch, exit_):
    # well-separated clusters: Lloyd reaches its fixed point within a few
    # iterations; stopping there (default) or running all 10 gives the
    # reference's assignment and centroid bits
    monkeypatch.setenv("LCN_LLOYD_EARLY_EXIT", exit_)
    x = rng_points(51, 30000, 16, comps=24, spread=40.0)
    c_gpu, a_gpu = lcn.lloyd(ctx, x, 24, 10, 51)
    c_ref, a_ref = ref.lloyd(x, 24, 10, 51)
    assert np.array_equal(a_gpu, a_ref)
    assert np.array_equal(c_gpu.view(np.uint64), c_ref.view(np.uint64))


def test_lloyd_tile_skipping_bit_exact(ctx, ref, monkeypatch):
    # >= 8 tiles of 128 centroids: after the first full assignment each
    # cluster of 256 (sorted) points evaluates only the tiles its bounds do
    # not exclude -- assignment and centroid bits equal to the reference and
    # to evaluating every tile
    r = np.random.default_rng(71)
    means = r.standard_normal((200, 32)) * 3.0
    x = (means[r.integers(0, 200, 100_000)] + 0.5 * r.standard_normal((100_000, 32))).astype(np.float32)
    x = x.astype(np.float64)
    c1, a1 = lcn.lloyd(ctx, x, 1024, 10, 71)
    c_ref, a_ref = ref.lloyd(x, 1024, 10, 71)
    assert np.array_equal(a1, a_ref)
    assert np.array_equal(c1.view(np.uint64), c_ref.view(np.uint64))
    monkeypatch.setenv("LCN_LLOYD_TILES", "0")
    c0, a0 = lcn.lloyd(ctx, x, 1024, 10, 71)
    assert np.array_equal(a0, a1)
    assert np.array_equal(c0.view(np.uint64), c1.view(np.uint64))
