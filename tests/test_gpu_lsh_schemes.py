"""GPU parity for the other LSH schemes of lsh_neighbor_pairs (lsh.cpp:55-143):
cross-polytope hashing and hierarchical k-means, through the C-ABI, against
the golden vectors (tests/golden, made by the reference itself) and the
reference compiled from its own sources (oracle/_ref). Bucket ids and the
resulting support are bit-exact.
"""
import json
import os

import numpy as np
import pytest

import paper_2107_06876_b200 as lcn

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
ARR = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def mixture(seed, n, d, comps=6):
    r = np.random.default_rng(seed)
    means = r.standard_normal((comps, d)) * 3
    return means[r.integers(0, comps, n)] + r.standard_normal((n, d))


def test_cross_polytope_hand_oracle(ctx):
    # test_lsh.cpp:16-27
    proj = np.zeros((2, 2))
    proj[0, 0] = proj[1, 1] = 1.0
    x = np.array([[1.0, 0.0], [-1.0, 0.0], [0.6, 0.8]])
    assert lcn.cross_polytope_buckets(ctx, x, proj).tolist() == [0, 2, 1]


def test_cross_polytope_ties_first_maximum(ctx):
    proj = np.array([[1.0, 1.0, 0.0]])
    x = np.array([[0.0], [2.0], [-2.0]])
    assert lcn.cross_polytope_buckets(ctx, x, proj).tolist() == [0, 0, 3]


@pytest.mark.parametrize("n,d,half,seed", [(5000, 37, 100, 1), (777, 5, 3, 2), (3000, 128, 256, 3), (70, 1, 65, 4)])
def test_cross_polytope_bit_exact(ctx, ref, n, d, half, seed):
    r = np.random.default_rng(seed)
    x = r.standard_normal((n, d))
    proj = r.standard_normal((d, half))
    if seed == 4:
        proj[:, 64] = proj[:, 0]  # equal columns across column tiles: exact ties
    assert np.array_equal(lcn.cross_polytope_buckets(ctx, x, proj), ref.cross_polytope_bucket(x, proj))


@pytest.mark.parametrize("key", [k for k in GOLD if k.startswith("lsh_")])
def test_lsh_schemes_golden(ctx, key):
    scheme, bands, rows, buckets, branching, seed = map(int, key.split("_")[1:])
    cfg = lcn.LshConfig(bands, rows, buckets, 10, seed, scheme, branching)
    ids = lcn.lsh_buckets(ctx, ARR["lsh_p"], ARR["lsh_q"], cfg)
    assert np.array_equal(ids, ARR[key + "_ids"].astype(np.uint64))


@pytest.mark.parametrize("scheme,bands,rows,buckets,branching,n,d", [
    (lcn.LSH_CROSS_POLYTOPE, 2, 2, 16, 2, 3000, 12),
    (lcn.LSH_CROSS_POLYTOPE, 1, 1, 512, 2, 20000, 64),
    (lcn.LSH_HIERARCHICAL_KMEANS, 1, 1, 64, 2, 4000, 8),
    (lcn.LSH_HIERARCHICAL_KMEANS, 2, 1, 30, 4, 3000, 16),
    (lcn.LSH_HIERARCHICAL_KMEANS, 1, 2, 8, 3, 2000, 5),
])
def test_lsh_schemes_vs_reference(ctx, ref, scheme, bands, rows, buckets, branching, n, d):
    p, q = mixture(n, n, d), mixture(n + 1, n // 2, d)
    cfg = lcn.LshConfig(bands, rows, buckets, 10, 99, scheme, branching)
    ids = lcn.lsh_buckets(ctx, p, q, cfg)
    assert np.array_equal(ids, ref.lsh_buckets_cfg(p, q, scheme, bands, rows, buckets, 10, branching, 99))


def test_cross_polytope_odd_buckets_rejected(ctx):
    p = mixture(1, 10, 3)
    with pytest.raises(lcn.InvalidArgument, match="even bucket count"):
        lcn.lsh_buckets(ctx, p, p, lcn.LshConfig(1, 1, 3, 10, 0, lcn.LSH_CROSS_POLYTOPE))


def test_hierarchical_four_clusters(ctx):
    # test_lsh.cpp:71-96
    r = np.random.default_rng(5)
    centers = np.array([[0, 0], [50, 0], [0, 50], [50, 50]], float)
    truth = np.arange(12) % 4
    x = centers[truth] + r.uniform(-0.2, 0.2, (12, 2))
    ids = lcn.lsh_buckets(ctx, x[:6], x[6:], lcn.LshConfig(1, 1, 4, 10, 9, lcn.LSH_HIERARCHICAL_KMEANS, 2))[0]
    assert len(set(ids.tolist())) == 4
    assert np.array_equal(ids[:, None] == ids[None, :], truth[:, None] == truth[None, :])


@pytest.mark.parametrize("scheme,bands,rows,buckets,branching", [(lcn.LSH_CROSS_POLYTOPE, 2, 1, 16, 2),
                                                                 (lcn.LSH_HIERARCHICAL_KMEANS, 1, 1, 24, 2)])
def test_sparse_operator_on_scheme(ctx, ref, scheme, bands, rows, buckets, branching):
    """lsh_neighbor_pairs -> build_sparse -> sinkhorn with the scheme's support."""
    x = mixture(11, 2700, 6)
    p, q = x[:1500], x[1500:]
    cfg = lcn.LshConfig(bands, rows, buckets, 10, 5, scheme, branching)
    lam = 2.0
    op = lcn.KernelOperator.sparse_lsh(ctx, p, q, lcn.EUCLIDEAN, lam, cfg)
    pairs = ref.lsh_pairs_cfg(p, q, scheme, bands, rows, buckets, 10, branching, 5)
    rop = ref.op_sparse(p, q, lcn.EUCLIDEAN, lam, pairs)
    rp, col, _ = op.export_csr(0)
    rrp, rcol, _ = rop.csr(0)
    assert np.array_equal(rp, rrp) and np.array_equal(col, rcol)
    pm, qm = np.full(1500, 1 / 1500), np.full(1200, 1 / 1200)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=40, check_support=False))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=40, check_support=False)
    assert rel(res.distance, rres.distance) <= 1e-4


@pytest.mark.parametrize("case", ["one_band_full", "one_band_short", "two_band_union_full", "two_band_short"])
def test_support_check_block_matching(ctx, ref, case):
    """sinkhorn.cpp:122-128 support warning: band-1 block matching sum_b
    min(n_b, m_b) decides one band exactly; a short multi-band bound falls
    back to the general matching. Warnings must equal the reference's."""
    n = m = 6
    r = np.random.default_rng(3)
    p, q = r.standard_normal((n, 2)), r.standard_normal((m, 2))
    if case == "one_band_full":
        ids_p, ids_q = np.array([[0, 0, 1, 1, 2, 2]]), np.array([[2, 1, 0, 0, 1, 2]])
    elif case == "one_band_short":
        ids_p, ids_q = np.array([[0, 0, 0, 1, 1, 2]]), np.array([[0, 1, 1, 1, 2, 2]])
    elif case == "two_band_union_full":
        ids_p = np.array([[0, 0, 0, 1, 1, 2], [5, 6, 7, 8, 9, 10]])
        ids_q = np.array([[0, 1, 1, 1, 2, 2], [11, 12, 7, 13, 14, 15]])
        ids_q[1] = [5, 12, 7, 8, 9, 10]
    else:
        ids_p = np.array([[0, 0, 0, 1, 1, 2], [3, 3, 3, 4, 4, 4]])
        ids_q = np.array([[0, 1, 1, 1, 2, 2], [5, 5, 5, 4, 4, 4]])
    ids_p, ids_q = ids_p.astype(np.uint64), ids_q.astype(np.uint64)
    op = lcn.KernelOperator.sparse_buckets(ctx, p, q, lcn.EUCLIDEAN, 1.0, ids_p, ids_q)
    pairs = ref.pairs_from_buckets(ids_p, ids_q, 16)
    rop = ref.op_sparse(p, q, lcn.EUCLIDEAN, 1.0, pairs)
    pm = qm = np.full(n, 1.0 / n)
    try:
        res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=5))
        nw = len(res.warnings)
    except lcn.StabilizationError:
        nw = None
    try:
        nw_ref = rop.sinkhorn(pm, qm, tol=0.0, max_iters=5).n_warnings
    except Exception:
        nw_ref = None
    assert nw == nw_ref
