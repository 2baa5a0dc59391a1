"""The bucket-sharded LCN solve on the GPU, ranks emulated
as host threads over an in-process loopback communicator (lcn_loopback_*):
every rank builds only its shard (owned band-0 buckets + halo points) with
the CUDA build kernels and runs the sharded iteration (band passes over the
local blocks, low-rank passes over the owned rows, one all-gather per
half-iteration); the all-gather is a host barrier plus device copies, so no
kernel waits on another rank's kernel on the shared device. The gathered
result must equal the single-rank solve of the same problem."""
import threading

import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import configs

pytestmark = pytest.mark.gpu


def _run_ranks(world, build, store64, pm, qm, opts):
    group = lcn.LoopbackGroup(world)
    out = [None] * world

    def rank(r):
        try:
            c = lcn.Context(0, store_fp64=store64)
            c.set_loopback(group, r)
            op = build(c)
            res = lcn.sinkhorn(op, pm, qm, opts)
            out[r] = dict(distance=res.distance, log_s=res.log_s.copy(), log_t=res.log_t.copy(),
                          row_marginal=res.row_marginal.copy(), iters=res.iters, nnz=op.nnz, stored=op.stored,
                          n=op.n, m=op.m)
            del res, op
            c.close()
        except Exception as e:  # noqa: BLE001 - surfaced below
            group.abort()
            out[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    errs = [o for o in out if isinstance(o, Exception)]
    primary = [e for e in errs if "another rank failed" not in str(e)]
    if errs:
        raise (primary or errs)[0]
    return out


def _compare(single, shards, rtol_d, atol_v):
    d0 = single.distance
    for o in shards:
        assert o["iters"] == single.iters
        assert abs(o["distance"] - d0) <= rtol_d * abs(d0), (o["distance"], d0)
        assert np.max(np.abs(o["log_s"] - single.log_s)) <= atol_v
        assert np.max(np.abs(o["log_t"] - single.log_t)) <= atol_v
        assert np.allclose(o["row_marginal"], single.row_marginal, rtol=1e3 * atol_v, atol=0)
    for o in shards[1:]:  # every rank returns the same whole-problem result
        assert o["distance"] == shards[0]["distance"]
        assert np.array_equal(o["log_s"], shards[0]["log_s"])


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("store64", [True, False])
def test_sharded_lsh_solve_matches_single(world, store64):
    """configs[3]-shaped (k-means LSH, 2 bands, squared L2 / mean): the LSH
    and landmarks are computed on every rank (bit-exact, so identical), the
    operator is sharded by band-0 bucket."""
    pr = configs.config3(0.01)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    pm, qm = pr.marginals()
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=40, check_support=False, want_plan=False)

    def build(c):
        return lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                          pr.landmark_seed)

    c0 = lcn.Context(0, store_fp64=store64)
    op = build(c0)
    single = lcn.sinkhorn(op, pm, qm, opts)
    shards = _run_ranks(world, build, store64, pm, qm, opts)
    for o in shards:
        assert o["nnz"] == op.nnz and o["n"] == pr.n and o["m"] == pr.m
    if world > 1:  # each rank stores a part of the blocks
        assert all(o["stored"] < op.stored for o in shards)
    _compare(single, shards, 1e-12 if store64 else 2e-6, 1e-9 if store64 else 2e-5)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_solve_with_halo_exchange(world):
    """Independent random bucket ids in the two bands: later-band buckets
    span ranks, so every half-iteration moves halo scalings between ranks
    (external ids through lcn_op_lcn_buckets, explicit landmarks)."""
    r = np.random.default_rng(9)
    n, m, d, l, buckets = 900, 800, 8, 24, 16
    p = r.normal(size=(n, d))
    q = r.normal(size=(m, d)) + 0.3
    ids_p = r.integers(0, buckets, (2, n)).astype(np.uint64)
    ids_q = r.integers(0, buckets, (2, m)).astype(np.uint64)
    lm = np.concatenate([p[:l // 2], q[:l // 2]])
    pm = np.full(n, 1.0 / n)
    qm = np.full(m, 1.0 / m)
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=30, check_support=False, want_plan=False)

    def build(c):
        return lcn.KernelOperator.lcn_buckets(c, p, q, lcn.SQEUCLIDEAN, 4.0, ids_p, ids_q, landmarks=lm,
                                              range_=buckets)

    c0 = lcn.Context(0, store_fp64=True)
    op = build(c0)
    single = lcn.sinkhorn(op, pm, qm, opts)
    plan = lcn.ShardPlan(ids_p.astype(np.uint32), ids_q.astype(np.uint32), buckets, l, world)
    assert sum(plan.info(k)["n_halo"] for k in range(world)) > 0
    shards = _run_ranks(world, build, True, pm, qm, opts)
    _compare(single, shards, 1e-12, 1e-9)


def test_sharded_operator_rejects_unsupported_calls():
    pr = configs.config3(0.005)
    cfg = lcn.LshConfig(pr.bands, 1, pr.buckets, pr.kmeans_iters, pr.lsh_seed)
    group = lcn.LoopbackGroup(1)
    c = lcn.Context(0)
    c.set_loopback(group, 0)
    op = lcn.KernelOperator.lcn_lsh(c, pr.p, pr.q, pr.cost, pr.lam_eff, cfg, pr.landmarks, lcn.LANDMARK_KMEANS,
                                    pr.landmark_seed)
    pm, qm = pr.marginals()
    with pytest.raises(lcn.InvalidArgument, match="want_plan"):
        lcn.sinkhorn(op, pm, qm, lcn.SinkhornOptions(tol=0.0, max_iters=3, want_plan=True))
    with pytest.raises(lcn.InvalidArgument, match="sharded"):
        op.export_csr(1)
    with pytest.raises(lcn.InvalidArgument, match="sharded"):
        op.log_matvec(np.zeros(pr.m))


@pytest.mark.parametrize("world", [3, 5])
def test_sharded_solve_with_idle_ranks(world):
    """More ranks than band-0 bucket groups: some ranks own no point at all
    and only take part in the exchanges; the result is unchanged."""
    r = np.random.default_rng(4)
    n, m, d = 300, 280, 6
    p = r.normal(size=(n, d))
    q = r.normal(size=(m, d)) + 0.2
    ids_p = np.stack([r.integers(0, 2, n), r.integers(0, 3, n)]).astype(np.uint64)
    ids_q = np.stack([r.integers(0, 2, m), r.integers(0, 3, m)]).astype(np.uint64)
    lm = np.concatenate([p[:5], q[:5]])
    pm = np.full(n, 1.0 / n)
    qm = np.full(m, 1.0 / m)
    opts = lcn.SinkhornOptions(tol=0.0, max_iters=25, check_support=False, want_plan=False)

    def build(c):
        return lcn.KernelOperator.lcn_buckets(c, p, q, lcn.SQEUCLIDEAN, 3.0, ids_p, ids_q, landmarks=lm, range_=3)

    plan = lcn.ShardPlan(ids_p.astype(np.uint32), ids_q.astype(np.uint32), 3, 10, world)
    assert any(plan.info(k)["n_own"] + plan.info(k)["m_own"] == 0 for k in range(world))
    c0 = lcn.Context(0, store_fp64=True)
    single = lcn.sinkhorn(build(c0), pm, qm, opts)
    shards = _run_ranks(world, build, True, pm, qm, opts)
    _compare(single, shards, 1e-12, 1e-9)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lloyd_bit_identical(world):
    """Lloyd with the assignments split over the ranks (rank r assigns
    points [r S, (r + 1) S), one all-gather per assignment): the tensor-core
    filter with certified bounds on each slice, the centroid update on every
    rank -- assignment and centroid bits equal to the single-rank Lloyd."""
    r = np.random.default_rng(61)
    means = r.standard_normal((150, 128))
    x = (means[r.integers(0, 150, 200_001)] + 0.5 * r.standard_normal((200_001, 128))).astype(np.float32)
    x = x.astype(np.float64)
    c0 = lcn.Context(0)
    ref_c, ref_a = lcn.lloyd(c0, x, 512, 10, 61)
    c0.close()
    group = lcn.LoopbackGroup(world)
    out = [None] * world

    def rank(rk):
        try:
            c = lcn.Context(0)
            c.set_loopback(group, rk)
            out[rk] = lcn.lloyd(c, x, 512, 10, 61)
            c.close()
        except Exception as e:  # noqa: BLE001 - surfaced below
            group.abort()
            out[rk] = e

    th = [threading.Thread(target=rank, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for o in out:
        if isinstance(o, Exception):
            raise o
        cc, aa = o
        assert np.array_equal(aa, ref_a)
        assert np.array_equal(cc.view(np.uint64), ref_c.view(np.uint64))
