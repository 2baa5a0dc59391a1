"""BP extension (KernelOperator::with_bp, operator.cpp:103-115 and 226-266;
the extended solve of sinkhorn.cpp:115-120) on the GPU against the reference,
for every operator kind: extended scalings, distance, trace, deletion masses."""
import numpy as np
import pytest

import paper_2107_06876_b200 as lcn

pytestmark = pytest.mark.gpu


def problem(seed=3, n=180, m=150, d=4):
    r = np.random.default_rng(seed)
    p = r.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    q = (r.standard_normal((m, d)) * 0.8 + 0.3).astype(np.float32).astype(np.float64)
    pm = r.uniform(0.5, 1.5, n)
    qm = r.uniform(0.5, 1.5, m)
    return p, q, pm / pm.sum(), 0.7 * qm / qm.sum()  # unbalanced: BP allows it


def build(ctx, ref, kind, p, q, lam):
    if kind == "dense":
        return lcn.KernelOperator.dense(ctx, p, q, lcn.EUCLIDEAN, lam), ref.op_dense(p, q, lcn.EUCLIDEAN, lam)
    cfg = lcn.LshConfig(1, 1, 6, 10, 11)
    pairs = ref.lsh_pairs(p, q, 1, 6, 10, 11)
    if kind == "sparse":
        return (lcn.KernelOperator.sparse_lsh(ctx, p, q, lcn.EUCLIDEAN, lam, cfg),
                ref.op_sparse(p, q, lcn.EUCLIDEAN, lam, pairs))
    return (lcn.KernelOperator.lcn_lsh(ctx, p, q, lcn.EUCLIDEAN, lam, cfg, 12, lcn.LANDMARK_KMEANS, 5),
            ref.op_lcn(p, q, lcn.EUCLIDEAN, lam, pairs, 12, 0, 5))


@pytest.mark.parametrize("fp64", [True, False])
@pytest.mark.parametrize("kind", ["dense", "sparse", "lcn"])
def test_bp_solve_matches_reference(ref, kind, fp64):
    p, q, pm, qm = problem()
    lam = 0.5
    r = np.random.default_rng(9)
    cp, cq = r.uniform(1.0, 3.0, len(pm)), r.uniform(1.0, 3.0, len(qm))
    ctx = lcn.Context(0, store_fp64=fp64)
    op, rop = build(ctx, ref, kind, p, q, lam)
    op.with_bp(cp, cq)
    rop.with_bp(cp, cq, lam)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=60))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=60)
    tol = 1e-9 if fp64 else 1e-4
    assert res.iters == rres.iters == 60
    assert abs(res.distance - rres.distance) <= tol * abs(rres.distance)
    assert np.allclose(res.log_s, rres.log_s, rtol=0, atol=tol * 10)
    assert np.allclose(res.log_t, rres.log_t, rtol=0, atol=tol * 10)
    # the trace reaches the storage-precision floor (fp32: ~1e-8 of the mass)
    assert np.allclose(res.marginal_err, rres.marginal_err, rtol=1e-3 if not fp64 else 1e-7, atol=1e-9 if fp64 else 2e-6)
    assert np.allclose(res.del_p_mass, rres.del_p_mass, rtol=tol * 10, atol=0)
    assert np.allclose(res.del_q_mass, rres.del_q_mass, rtol=tol * 10, atol=0)
    assert abs(res.eps_mass - rres.eps_mass) <= tol * 10 * abs(rres.eps_mass)


def test_bp_converges_and_rejects_bad_kernels(ref):
    p, q, pm, qm = problem(5, 90, 70)
    ctx = lcn.Context(0, store_fp64=True)
    op, rop = build(ctx, ref, "dense", p, q, 0.3)
    op.with_bp(np.full(90, 1.5), np.full(70, 1.5))
    rop.with_bp(np.full(90, 1.5), np.full(70, 1.5), 0.3)
    res = lcn.sinkhorn(op, pm, qm)  # default tol 1e-6 * total mass
    rres = rop.sinkhorn(pm, qm, tol=-1.0, max_iters=500)
    assert res.converged == rres.converged and res.iters == rres.iters
    with pytest.raises(lcn.InvalidArgument, match="deletion kernels must be finite and nonnegative"):
        op.with_bp(np.full(90, np.nan), np.full(70, 1.0))


@pytest.mark.parametrize("kind", ["dense", "lcn"])
def test_bp_grad_cost_rejected(ref, kind):
    # grad_cost on a BP-extended operator throws InvalidArgument after the
    # stale warning (sinkhorn.cpp:265-270), like the reference
    p, q, pm, qm = problem(7, 60, 50)
    ctx = lcn.Context(0, store_fp64=True)
    op, rop = build(ctx, ref, kind, p, q, 0.5)
    op.with_bp(np.full(60, 1.2), np.full(50, 1.2))
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=5))
    for which in ((0,) if kind == "dense" else (1, 2, 3)):
        with pytest.raises(lcn.InvalidArgument, match="gradients are defined for the unextended operators"):
            lcn.grad_cost(res, op, which)


def test_bp_device_solve_rejected(ref):
    # the device-marginal entry solves only the balanced base problem: a BP
    # operator must go through lcn_sinkhorn, not be solved unextended silently
    import torch
    p, q, pm, qm = problem(8, 40, 30)
    ctx = lcn.Context(0, store_fp64=True)
    op, _ = build(ctx, ref, "sparse", p, q, 0.5)
    op.with_bp(np.full(40, 1.0), np.full(30, 1.0))
    dp = torch.from_numpy(pm).cuda()
    dq = torch.from_numpy(qm).cuda()
    with pytest.raises(lcn.InvalidArgument, match="BP-extended"):
        lcn.sinkhorn_device(op, dp.data_ptr(), dq.data_ptr(), lcn.SinkhornOptions(tol=0.0, max_iters=5))


def test_bp_sparse_skips_support_check(ref):
    # sinkhorn.cpp:122: the support check runs only without BP, so a BP solve
    # of a pattern without support emits no warning
    p, q, pm, qm = problem(9, 70, 40)
    ctx = lcn.Context(0, store_fp64=True)
    op, rop = build(ctx, ref, "sparse", p, q, 0.5)
    op.with_bp(np.full(70, 1.0), np.full(40, 1.0))
    rop.with_bp(np.full(70, 1.0), np.full(40, 1.0), 0.5)
    res = lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=5, check_support=True))
    rres = rop.sinkhorn(pm, qm, tol=0.0, max_iters=5, check_support=True)
    assert len(res.warnings) == rres.n_warnings == 0
