"""CPU suite (no GPU): the oracle pinned against the reference's golden vectors
and known answers, the host logic, and the C-ABI library's exports.

Golden vectors: tests/golden/golden.{json,npz}, produced by
tests/golden/make_golden.py from the reference's own sources compiled
unmodified (oracle/_ref). Known answers: the reference's unit tests
(test_sinkhorn.cpp, test_sparse.cpp, test_nystrom.cpp, test_lsh.cpp).
"""
import ctypes
import hashlib
import json
import math
import os
import re

import numpy as np
import pytest

from oracle.bindings import LcnError, OracleLib, RefLib, oracle_available, ref_available
from paper_2107_06876_b200 import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
ARR = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))

pytestmark = pytest.mark.skipif(not oracle_available(), reason="oracle not built (make -C oracle oracle)")


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def ball(n, d, seed):
    return ARR[f"ball_{n}_{d}_{seed}"]


# ---------------------------------------------------------------------------
# golden vectors from the reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("key,make", [("c0", lambda: configs.config0()), ("c1s", lambda: configs.config1(0.05)),
                                      ("c3s", lambda: configs.config3(0.002))])
def test_golden_configs(orc, key, make):
    g = GOLD[key]
    pr = make()
    assert sha(pr.p, pr.q) == g["points_sha256"], "synthetic generator drifted"
    assert pr.lam_eff == g["lam_eff"]
    ids = orc.lsh_buckets(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    assert np.array_equal(ids, ARR[f"{key}_ids"].astype(np.uint64))  # bucket ids bit-exact
    pairs = orc.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    if pr.landmarks:
        op = orc.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, pairs, pr.landmarks, 0, pr.landmark_seed)
    else:
        op = orc.op_sparse(pr.p, pr.q, pr.cost, pr.lam_eff, pairs)
    rp, col, logk = op.csr(0)
    assert sha(rp, col) == g["support_sha256"]                         # support bit-exact
    assert sha(logk) == g["logk_sha256"]                               # log K bit-exact
    pm, qm = pr.marginals()
    res = op.sinkhorn(pm, qm, tol=0.0, max_iters=pr.iters)
    assert res.iters == g["iters"] and res.n_warnings == g["warnings"]
    assert rel(res.distance, g["distance"]) <= 1e-12
    plan = res.sp_vals if pr.landmarks else res.sparse_vals
    assert rel(plan[ARR[f"{key}_plan_idx"]], ARR[f"{key}_plan"]) <= 1e-12
    assert rel(res.log_s[:: max(1, pr.n // 64)], ARR[f"{key}_log_s"]) <= 1e-12
    if pr.landmarks:
        assert rel(res.distance_lcn(), g["distance_lcn"]) <= 1e-12


@pytest.mark.parametrize("key", [k for k in GOLD if k.startswith("lloyd_")])
def test_golden_lloyd(orc, key):
    _, n, d, k, seed = key.split("_")
    x = ARR[key + "_x"]
    ctr, asg = orc.lloyd(x, int(k), 10, int(seed))
    assert np.array_equal(asg, ARR[key + "_assign"])
    assert sha(ctr) == GOLD[key]["centroids_sha256"]
    assert orc.kmeans_pp(x, int(k), int(seed)).tolist() == GOLD[key]["pp"]


def test_mt19937_64_check_value(orc):
    # C++ [rand.predef]: the 10000th consecutive invocation of a default-constructed
    # mt19937_64 (seed 5489) produces 9981545732273789042.
    lib = orc.lib
    lib.orc_mt19937_64_nth.restype = ctypes.c_uint64
    lib.orc_mt19937_64_nth.argtypes = [ctypes.c_uint64, ctypes.c_size_t]
    assert lib.orc_mt19937_64_nth(5489, 9999) == 9981545732273789042
    from paper_2107_06876_b200.native import _MT19937_64
    g = _MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_uniform_index_matches_host_mirror(orc):
    from paper_2107_06876_b200.native import _MT19937_64, _lemire
    lib = orc.lib
    lib.orc_uniform_index.restype = ctypes.c_uint64
    lib.orc_uniform_index.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    for seed, n in [(1, 7), (99, 1000003), (2**63 + 5, 2**40 + 3), (7, 1)]:
        assert lib.orc_uniform_index(seed, n) == _lemire(_MT19937_64(seed), n)


# ---------------------------------------------------------------------------
# oracle vs the compiled reference, edge cases
# ---------------------------------------------------------------------------
needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("n,d,k,seed,dup", [(30, 2, 30, 3, False), (50, 3, 7, 8, True), (200, 5, 9, 1, False)])
def test_oracle_kmeans_vs_reference(orc, n, d, k, seed, dup):
    r = np.random.default_rng(seed)
    x = r.standard_normal((n, d))
    if dup:
        x[: n // 2] = x[0]  # many coincident points: total <= 0 and reseeding paths
    ref = RefLib()
    c1, a1 = orc.lloyd(x, k, 10, seed)
    c2, a2 = ref.lloyd(x, k, 10, seed)
    assert np.array_equal(a1, a2) and np.array_equal(c1.view(np.uint64), c2.view(np.uint64))
    assert np.array_equal(orc.kmeans_pp(x, k, seed), ref.kmeans_pp(x, k, seed))


@needs_ref
@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_oracle_cost_kinds_vs_reference(orc, kind):
    p, q = ball(20, 3, 900) + 0.1, ball(20, 3, 901) + 0.1
    ref = RefLib()
    pr_o = orc.lsh_pairs(p, q, 2, 3, 10, 77)
    pr_r = ref.lsh_pairs(p, q, 2, 3, 10, 77)
    assert all(np.array_equal(a, b) for a, b in zip(pr_o.arrays(), pr_r.arrays()))
    lam = 0.5 if kind != 1 else 5.0
    oo, orr = orc.op_sparse(p, q, kind, lam, pr_o), ref.op_sparse(p, q, kind, lam, pr_r)
    assert np.array_equal(oo.csr(0)[2].view(np.uint64), orr.csr(0)[2].view(np.uint64))
    pm = np.full(20, 0.05)
    ro, rr = oo.sinkhorn(pm, pm, tol=0.0, max_iters=30), orr.sinkhorn(pm, pm, tol=0.0, max_iters=30)
    assert rel(ro.distance, rr.distance) <= 1e-13


# ---------------------------------------------------------------------------
# known answers from the reference's unit tests, through the oracle
# ---------------------------------------------------------------------------
def test_one_by_one_forced_in_one_sweep(orc):
    # test_sinkhorn.cpp:64-74
    op = orc.op_dense(np.array([[0.0]]), np.array([[2.5]]), 0, 0.8)
    res = op.sinkhorn(np.array([1.0]), np.array([1.0]))
    assert res.iters == 1 and res.converged
    assert res.distance == pytest.approx(2.5, rel=1e-12)


def test_two_by_two_zero_cost_is_minus_ln4(orc):
    # test_sinkhorn.cpp:76-88
    x = np.array([[0.3], [0.3]])
    res = orc.op_dense(x, x, 0, 1.0).sinkhorn(np.full(2, 0.5), np.full(2, 0.5))
    assert res.distance == pytest.approx(-math.log(4.0), rel=1e-12)


def test_dense_matches_serial_linear_reference(orc):
    # test_sinkhorn.cpp:90-114 (independent serial solver, reference.cpp:41-105)
    r = np.random.default_rng(101)
    for rep in range(3):
        p, q = ball(20, 3, 900)[:6], ball(20, 3, 901)[:6]
        pm = r.uniform(0.2, 1.0, 6)
        qm = r.uniform(0.2, 1.0, 6)
        pm, qm = pm / pm.sum(), qm / qm.sum()
        qm *= pm.sum() / qm.sum()
        lam = 0.5 if rep % 2 == 0 else 0.1
        res = orc.op_dense(p, q, 0, lam).sinkhorn(pm, qm, tol=1e-10, max_iters=100000)
        cost = np.sqrt(((p[:, None, :] - q[None, :, :]) ** 2).sum(-1))
        _, dist, _ = orc.dense_reference(cost, pm, qm, lam, 1e-10, 100000)
        assert res.converged
        assert res.distance == pytest.approx(dist, rel=1e-8)


def test_equidistant_pair_closed_form(orc):
    # test_nystrom.cpp:110-119: K_Nys = 2 e^-2 / (1 + e^-2) = 0.23841
    z = np.zeros((1, 2))
    op = orc.op_lcn(z, z, 0, 1.0, None, 2, landmarks=np.array([[-1.0, 0.0], [1.0, 0.0]]), nystrom_only=True)
    u, w = op.dense_factor(2), op.dense_factor(3)
    closed = 2.0 * math.exp(-2.0) / (1.0 + math.exp(-2.0))
    assert (u @ w)[0, 0] == pytest.approx(closed, rel=1e-12)
    assert closed == pytest.approx(0.23841, rel=1e-4)


def test_single_landmark_rank_one(orc):
    # test_nystrom.cpp:81-94
    p, q = ball(4, 2, 11), ball(3, 2, 12)
    lm = np.array([[0.25, -0.1]])
    op = orc.op_lcn(p, q, 0, 0.7, None, 1, landmarks=lm, nystrom_only=True)
    ki = np.exp(-np.linalg.norm(p - lm, axis=1) / 0.7)
    kj = np.exp(-np.linalg.norm(q - lm, axis=1) / 0.7)
    assert rel(op.dense_factor(2) @ op.dense_factor(3), np.outer(ki, kj)) <= 1e-12


def test_duplicate_landmarks_survive_via_jitter(orc):
    # test_nystrom.cpp:190-197
    p, q = ball(8, 3, 22)[:, :2], ball(8, 3, 23)[:, :2]
    lm = np.array([[0.1, 0.2], [0.1, 0.2], [-0.3, 0.4]])
    op = orc.op_lcn(p, q, 0, 0.5, None, 3, landmarks=lm, nystrom_only=True)
    assert np.all(np.isfinite(op.dense_factor(3)))
    assert op.scalar(1) > 1.0


def test_identity_pattern_acts_as_identity(orc):
    # test_sparse.cpp:129-137
    x = ball(3, 2, 12)[:2]
    pairs = orc.pairs_from_arrays(2, 2, [0, 1], [0, 1])
    op = orc.op_sparse(x, x, 0, 1.0, pairs)
    out = op.log_matvec(np.log([2.0, 3.0]))
    assert np.exp(out) == pytest.approx([2.0, 3.0], rel=1e-15)


def test_empty_pattern_is_zero_operator(orc):
    # test_sparse.cpp:74-81
    pairs = orc.pairs_from_arrays(6, 5, [], [])
    op = orc.op_sparse(ball(6, 3, 1), ball(5, 3, 2), 0, 0.4, pairs)
    assert np.all(op.log_matvec(np.zeros(5)) == -np.inf)


def test_lcn_collapses_to_dense_with_full_pattern(orc):
    # test_sinkhorn.cpp:196-206: a full pattern corrects any landmark choice
    p, q = ball(12, 2, 1000), ball(12, 2, 1001)
    pm = np.full(12, 1 / 12)
    dense = orc.op_dense(p, q, 0, 0.4).sinkhorn(pm, pm, tol=1e-10, max_iters=50000)
    full = orc.pairs_from_arrays(12, 12, np.repeat(np.arange(12), 12), np.tile(np.arange(12), 12))
    op = orc.op_lcn(p, q, 0, 0.4, full, 3, 0, 6)
    res = op.sinkhorn(pm, pm, tol=1e-10, max_iters=50000)
    assert res.distance == pytest.approx(dense.distance, rel=1e-8)
    assert res.distance_lcn() == pytest.approx(dense.distance, rel=1e-8)


def test_empty_row_is_stabilization_error_naming_sparse(orc):
    # test_sinkhorn.cpp:241-248
    p, q = ball(3, 2, 1100), ball(3, 2, 1101)
    pairs = orc.pairs_from_arrays(3, 3, [0, 2, 2], [0, 1, 2])
    op = orc.op_sparse(p, q, 0, 0.5, pairs)
    with pytest.raises(LcnError) as e:
        op.sinkhorn(np.full(3, 1 / 3), np.full(3, 1 / 3), check_support=False)
    assert e.value.kind == "StabilizationError" and "sparse" in e.value.msg


def test_no_support_warns_and_iterates(orc):
    # test_sinkhorn.cpp:229-240
    p, q = ball(3, 2, 1100), ball(3, 2, 1101)
    pairs = orc.pairs_from_arrays(3, 3, [0, 1, 2, 2], [0, 0, 1, 2])
    res = orc.op_sparse(p, q, 0, 0.5, pairs).sinkhorn(np.full(3, 1 / 3), np.full(3, 1 / 3), max_iters=50)
    assert res.n_warnings == 1 and not res.converged and math.isfinite(res.distance)


def test_band_or_semantics(orc):
    # test_lsh.cpp:98-126
    pairs = orc.pairs_from_buckets(np.array([[0], [5]], np.uint64), np.array([[1], [5]], np.uint64), 6)
    rows, cols = pairs.arrays()
    assert rows.tolist() == [0] and cols.tolist() == [0]
    pairs = orc.pairs_from_buckets(np.array([[7, 7, 7]], np.uint64), np.array([[7, 7]], np.uint64), 8)
    assert len(pairs.arrays()[0]) == 6


def test_kmeans_k_equals_n_and_too_many_buckets(orc):
    # test_lsh.cpp:59-69
    x = np.random.default_rng(2).uniform(size=(5, 2))
    _, a = orc.lloyd(x, 5, 10, 0)
    assert len(set(a.tolist())) == 5
    with pytest.raises(LcnError) as e:
        orc.lloyd(x, 6, 10, 0)
    assert e.value.kind == "InvalidArgument"


# ---------------------------------------------------------------------------
# the other LSH schemes: cross-polytope and hierarchical k-means (lsh.cpp:55-143)
# ---------------------------------------------------------------------------
def test_cross_polytope_hand_oracle(orc):
    # test_lsh.cpp:16-27: identity columns, d=2, b=4 -> (x0, x1, -x0, -x1)
    proj = np.zeros((2, 2))
    proj[0, 0] = proj[1, 1] = 1.0
    x = np.array([[1.0, 0.0], [-1.0, 0.0], [0.6, 0.8]])
    assert orc.cross_polytope_bucket(x, proj).tolist() == [0, 2, 1]


def test_cross_polytope_first_maximum_wins(orc):
    # ties: v == -v at 0 and equal columns -> the lowest concatenated index
    proj = np.array([[1.0, 1.0, 0.0]])
    x = np.array([[0.0], [2.0], [-2.0]])
    assert orc.cross_polytope_bucket(x, proj).tolist() == [0, 0, 3]


@pytest.mark.parametrize("seed", [0, 7, 2024])
def test_normal_draws_golden(orc, seed):
    # std::normal_distribution<double> over mt19937_64 (libstdc++ polar method)
    assert np.array_equal(orc.normal_draws(seed, 33).view(np.uint64), ARR[f"normal_{seed}"].view(np.uint64))


@pytest.mark.parametrize("key", [k for k in GOLD if k.startswith("lsh_")])
def test_golden_lsh_schemes(orc, key):
    scheme, bands, rows, buckets, branching, seed = map(int, key.split("_")[1:])
    p, q = ARR["lsh_p"], ARR["lsh_q"]
    ids = orc.lsh_buckets_cfg(p, q, scheme, bands, rows, buckets, 10, branching, seed)
    assert np.array_equal(ids, ARR[key + "_ids"].astype(np.uint64))
    assert int(ids.max()) == GOLD[key]["max_id"]
    if "pairs_sha256" in GOLD[key]:  # in-range ids only (see make_golden.py)
        n = p.shape[0]
        pairs = orc.pairs_from_buckets(ids[:, :n], ids[:, n:], 0)
        assert sha(*pairs.arrays()) == GOLD[key]["pairs_sha256"]
        assert GOLD[key]["nnz"] > 0


def test_cross_polytope_odd_buckets_rejected(orc):
    # test_lsh.cpp:29-35
    p = ball(10, 4, 41)
    with pytest.raises(LcnError) as e:
        orc.lsh_buckets_cfg(p, p, 0, 1, 1, 3, 10, 2, 0)
    assert e.value.kind == "InvalidArgument"


def test_hierarchical_recovers_four_clusters(orc):
    # test_lsh.cpp:71-96: four tight clusters, branching 2, buckets 4
    r = np.random.default_rng(5)
    centers = np.array([[0, 0], [50, 0], [0, 50], [50, 50]], float)
    truth = np.arange(12) % 4
    x = centers[truth] + r.uniform(-0.2, 0.2, (12, 2))
    ids = orc.lsh_buckets_cfg(x[:6], x[6:], 2, 1, 1, 4, 10, 2, 9)[0]
    assert len(set(ids.tolist())) == 4
    assert np.array_equal(ids[:, None] == ids[None, :], truth[:, None] == truth[None, :])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("scheme,bands,rows,buckets,branching", [(0, 2, 2, 8, 2), (0, 1, 1, 64, 2), (2, 1, 1, 24, 2),
                                                                 (2, 1, 1, 20, 5), (2, 1, 1, 19, 3), (1, 2, 2, 6, 2)])
def test_oracle_lsh_schemes_vs_reference(orc, scheme, bands, rows, buckets, branching):
    r = np.random.default_rng(buckets)
    p, q = r.standard_normal((300, 7)), r.standard_normal((250, 7)) + 0.5
    ref = RefLib()
    a = orc.lsh_buckets_cfg(p, q, scheme, bands, rows, buckets, 10, branching, 11)
    b = ref.lsh_buckets_cfg(p, q, scheme, bands, rows, buckets, 10, branching, 11)
    assert np.array_equal(a, b)
    if a.max() >= buckets ** rows:
        return  # leaves overshot buckets_per_fn: the reference's pair grouping is out of range
    n = p.shape[0]
    ra, ca = orc.pairs_from_buckets(a[:, :n], a[:, n:], 0).arrays()
    rb, cb = ref.lsh_pairs_cfg(p, q, scheme, bands, rows, buckets, 10, branching, 11).arrays()
    assert np.array_equal(ra, rb) and np.array_equal(ca, cb)


# ---------------------------------------------------------------------------
# boundary: the C-ABI library loads and exports every declared symbol
# ---------------------------------------------------------------------------
def test_capi_library_exports_header_symbols():
    import paper_2107_06876_b200 as lcn
    lib = lcn.library()
    header = open(os.path.join(ROOT, "include", "lcn_b200.h")).read()
    names = sorted(set(re.findall(r"\b(lcn_[a-z0-9_]+)\s*\(", header)))
    assert len(names) >= 25
    missing = [nm for nm in names if not hasattr(lib, nm)]
    assert not missing, missing
    assert lib.lcn_abi_version() == 5


def test_capi_without_gpu_fails_loudly():
    import paper_2107_06876_b200 as lcn
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(lcn.CudaError):
        lcn.Context(0)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_blocked_correction_bit_exact(monkeypatch):
    """oracle/ref_shims/correction_blocked.cpp (the full-size parity run's
    build_correction) gives the reference's build_correction bits
    (sparse_kernel.cpp:82-117): delta, nys_vals, the support and max |delta|,
    on a two-band k-means LSH pattern with buckets of uneven size."""
    from oracle.bindings import RefLib
    ref = RefLib()
    pr = configs.config3(0.002)
    ids = ref.lsh_buckets(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    lm = ref.select_landmarks(pr.p, pr.q, 40, configs.LANDMARK_KMEANS, pr.landmark_seed)
    ids_p, ids_q = np.ascontiguousarray(ids[:, :pr.n]), np.ascontiguousarray(ids[:, pr.n:])
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("LCN_REF_BLOCKED_CORRECTION", flag)
        op, _ = ref.lcn_pipeline(pr.p, pr.q, pr.cost, pr.lam_eff, ids_p, ids_q, pr.buckets, lm)
        out[flag] = [op.csr(1), op.csr(5), op.scalar(0)]
    (rp0, c0, d0), (_, _, n0), s0 = out["0"]
    (rp1, c1, d1), (_, _, n1), s1 = out["1"]
    assert len(c0) > 1000
    assert np.array_equal(rp0, rp1) and np.array_equal(c0, c1)
    assert np.array_equal(d0.view(np.uint64), d1.view(np.uint64))
    assert np.array_equal(n0.view(np.uint64), n1.view(np.uint64))
    assert s0 == s1
