"""The staged drop-in API: the reference's caller builds an
operator stage by stage and passes host structs between the stages
(runner.cpp:258-271: lsh_neighbor_pairs -> build_sparse -> select_landmarks
-> build_factors -> build_correction -> KernelOperator::lcn). Each stage here
runs on the GPU through the C-ABI and is checked against the same stage of
the compiled reference on the same inputs; the operator factories
(operator.hpp:33-36) take any CSR pattern, so the reference's own small
hand-built cases (test_sinkhorn.cpp:224-268) run through them too."""
import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0


def _csr_from_pairs(n, rows, cols):
    rp = np.zeros(n + 1, np.uint32)
    np.add.at(rp, rows.astype(np.int64) + 1, 1)
    return np.cumsum(rp).astype(np.uint32), cols.astype(np.uint32)


@pytest.mark.parametrize("fp64", [True, False])
def test_staged_lcn_pipeline_matches_reference(ref, fp64):
    pr = configs.config3(0.003)
    c = lcn.Context(0, store_fp64=fp64)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    # lsh_neighbor_pairs: the pattern, bit-exact
    rp, col = lcn.lsh_neighbor_pairs(c, pr.p, pr.q, cfg)
    rpairs = ref.lsh_pairs(pr.p, pr.q, pr.bands, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    rrows, rcols = rpairs.arrays()
    rrp, rcol = _csr_from_pairs(pr.n, rrows, rcols)
    assert len(col) > 1000 and np.array_equal(rp, rrp) and np.array_equal(col, rcol)
    # build_sparse: log K bit-exact
    lv = lcn.build_sparse(c, pr.p, pr.q, rp, col, pr.cost, pr.lam_eff)
    rs = ref.op_sparse(pr.p, pr.q, pr.cost, pr.lam_eff, rpairs)
    assert np.array_equal(lv.view(np.uint64), rs.csr(0)[2].view(np.uint64))
    # select_landmarks: bit-exact
    L = lcn.select_landmarks(c, pr.p, pr.q, pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
    rL = ref.select_landmarks(pr.p, pr.q, pr.landmarks, lcn.LANDMARK_KMEANS, pr.landmark_seed)
    assert np.array_equal(L.view(np.uint64), rL.view(np.uint64))
    # build_factors (restated Nystrom: long-double LDL^T, same jitter schedule)
    U, W, cond = lcn.build_factors(c, pr.p, pr.q, L, pr.cost, pr.lam_eff)
    rop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, rpairs, pr.landmarks, 0, pr.landmark_seed)
    assert rel(U, rop.dense_factor(2)) <= 1e-13
    assert np.max(np.abs(W - rop.dense_factor(3))) <= 1e-8 * max(1.0, np.max(np.abs(W)))
    # build_correction from the GPU stages' structs
    dl, nys, mx = lcn.build_correction(c, rp, col, lv, U, W)
    assert np.max(np.abs(dl - rop.csr(1)[2])) <= 1e-8
    assert np.max(np.abs(nys - rop.csr(5)[2])) <= 1e-8
    assert abs(mx - rop.scalar(0)) <= 1e-8
    # KernelOperator::lcn(factors, correction) -> sinkhorn
    op = lcn.KernelOperator.from_lcn(c, U, W, pr.lam_eff, rp, col, dl, lv, mx)
    assert op.kind() == "lcn" and op.nnz == len(col)
    pm, qm = pr.marginals()
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=60))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=60)
    tol = 1e-9 if fp64 else 1e-4
    assert rel(res.distance, rres.distance) <= tol
    assert rel(res.sp_vals, rres.sp_vals) <= tol
    assert rel(lcn.distance_lcn(res, op), rres.distance_lcn()) <= tol
    # KernelOperator::sparse(SparseKernel) and ::nystrom(NystromFactors)
    sop = lcn.KernelOperator.from_sparse(c, pr.n, pr.m, rp, col, lv, pr.lam_eff)
    sres = lcn.sinkhorn(sop, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=60, check_support=False))
    srres = rs.sinkhorn(pm, qm, tol=0.0, max_iters=60, check_support=False)
    assert rel(sres.distance, srres.distance) <= 1e-9
    nop = lcn.KernelOperator.from_nystrom(c, U, W, pr.lam_eff)
    nres = lcn.sinkhorn(nop, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=60))
    rnop = ref.op_lcn(pr.p, pr.q, pr.cost, pr.lam_eff, rpairs, pr.landmarks, 0, pr.landmark_seed, nystrom_only=True)
    assert rel(nres.distance, rnop.sinkhorn(pm, qm, tol=0.0, max_iters=60).distance) <= tol
    # log_matvec through the general-pattern operator
    lt = np.random.default_rng(1).normal(size=pr.m)
    assert rel(op.log_matvec(lt), rop.log_matvec(lt)) <= tol


def test_staged_dense_factory_matches_reference(ref, ctx64):
    r = np.random.default_rng(4)
    p = r.standard_normal((60, 5))
    q = r.standard_normal((50, 5)) + 0.2
    rop = ref.op_dense(p, q, lcn.EUCLIDEAN, 0.5)
    op = lcn.KernelOperator.from_dense_logk(ctx64, rop.dense_logk(), 0.5)
    pm, qm = np.full(60, 1 / 60), np.full(50, 1 / 50)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=80))
    assert rel(res.distance, rop.sinkhorn(pm, qm, tol=0.0, max_iters=80).distance) <= 1e-12


def test_reference_hand_built_cases(ref, ctx64):
    """test_sinkhorn.cpp:224-268 through the factories: a pattern without
    support only warns; an empty row is a StabilizationError naming the
    variant; a negative Nystrom product is a NegativeKernelError."""
    p = np.array([[0.1, 0.2], [0.5, -0.3], [-0.4, 0.4]])
    q = np.array([[0.0, 0.1], [0.3, 0.3], [-0.2, -0.5]])
    m3 = np.full(3, 1 / 3)
    rows, cols = np.array([0, 1, 2, 2]), np.array([0, 0, 1, 2])
    rp, col = _csr_from_pairs(3, rows, cols)
    lv = lcn.build_sparse(ctx64, p, q, rp, col, lcn.EUCLIDEAN, 0.5)
    op = lcn.KernelOperator.from_sparse(ctx64, 3, 3, rp, col, lv, 0.5)
    res = lcn.sinkhorn(op, m3, m3, lcn.SinkhornOptions(max_iters=50))
    assert res.warnings and "no support" in res.warnings[0]
    assert not res.converged and np.isfinite(res.distance)
    rows, cols = np.array([0, 2, 2]), np.array([0, 1, 2])
    rp, col = _csr_from_pairs(3, rows, cols)
    lv = lcn.build_sparse(ctx64, p, q, rp, col, lcn.EUCLIDEAN, 0.5)
    op = lcn.KernelOperator.from_sparse(ctx64, 3, 3, rp, col, lv, 0.5)
    with pytest.raises(lcn.StabilizationError, match="sparse"):
        lcn.sinkhorn(op, m3, m3, lcn.SinkhornOptions(check_support=False))
    # NystromFactors u = [[1], [1]], w = [[-2, 1]], empty correction
    U = np.ones((2, 1))
    W = np.array([[-2.0, 1.0]])
    op = lcn.KernelOperator.from_lcn(ctx64, U, W, 1.0, np.zeros(3, np.uint32), np.zeros(0, np.uint32), np.zeros(0),
                                     np.zeros(0))
    with pytest.raises(lcn.NegativeKernelError):
        lcn.sinkhorn(op, np.full(2, 0.5), np.full(2, 0.5))
    with pytest.raises(lcn.InvalidArgument, match="lambda must be positive"):
        lcn.KernelOperator.from_sparse(ctx64, 3, 3, rp, col, lv, 0.0)
    with pytest.raises(lcn.DimensionError):
        lcn.build_correction(ctx64, rp, col[:-1], lv[:-1], np.ones((3, 1)), np.ones((1, 3)))


def test_factorization_error_beyond_jitter_budget(ctx64):
    """build_factors (nystrom.cpp:104-124): a landmark kernel matrix that no
    jitter level makes factorizable (non-finite landmark coordinates) raises
    FactorizationError with the reference's message, through the staged API
    and through a configs[3]-sized operator build with external landmarks."""
    r = np.random.default_rng(3)
    p = r.normal(size=(50, 4))
    q = r.normal(size=(40, 4))
    L = r.normal(size=(6, 4))
    L[2, 1] = np.nan
    with pytest.raises(lcn.FactorizationError, match="jitter budget"):
        lcn.build_factors(ctx64, p, q, L, lcn.SQEUCLIDEAN, 1.0)
    pr = configs.config3(0.01)
    ids = lcn.lsh_kmeans_buckets(ctx64, pr.p, pr.q, lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters,
                                                                     pr.lsh_seed))
    Lbig = np.ascontiguousarray(pr.p[:pr.landmarks].copy())
    Lbig[5, 7] = np.inf
    with pytest.raises(lcn.FactorizationError):
        lcn.KernelOperator.lcn_buckets(ctx64, pr.p, pr.q, pr.cost, pr.lam_eff, ids[:, :pr.n], ids[:, pr.n:],
                                       landmarks=Lbig, range_=pr.buckets)
