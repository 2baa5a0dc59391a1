"""GPU parity for configs[4] (batched small LCN problems):
every problem of a seeded batch through the ragged launches of
lcn_batched_lcn against the reference pipeline run per problem
(oracle/_ref: lsh_neighbor_pairs -> build_sparse -> select_landmarks ->
build_factors -> build_correction -> KernelOperator::lcn -> sinkhorn).
Distances within 1e-9 relative (fp64 throughout); statuses (the
reference's errors) equal.
"""
import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from oracle.bindings import LcnError
from paper_2107_06876_b200 import configs

pytestmark = pytest.mark.gpu

STATUS = {"InvalidArgument": 2, "StabilizationError": 3, "NegativeKernelError": 4, "FactorizationError": 5}


def reference(ref, b, k):
    p, q = b.problem(k)
    try:
        return ref.lcn_problem(p, q, b.cost, b.lam, b.buckets, b.kmeans_iters, b.lsh_seed(k), b.landmarks,
                               b.landmark_seed(k), b.iters), 0
    except LcnError as e:
        return float("nan"), STATUS.get(e.kind, 6)


@pytest.mark.parametrize("scale", [8 / 4096])
def test_batched_matches_reference(ctx, ref, scale):
    b = configs.config4(scale)
    dist, st, it = lcn.batched_lcn(ctx, b)
    ok = 0
    for k in range(b.count):
        rd, rs = reference(ref, b, k)
        assert st[k] == rs, (k, st[k], rs)
        if rs == 0:
            ok += 1
            assert abs(dist[k] - rd) <= 1e-9 * abs(rd), (k, dist[k], rd)
            assert it[k] == b.iters
    assert ok > 0


def test_batched_variants(ctx, ref):
    """squared-L2 cost, more buckets and landmarks, sizes at the path's limits"""
    import dataclasses
    b = configs.config4(2 / 4096)
    b = dataclasses.replace(b, cost=configs.SQEUCLIDEAN, lam=2.0, buckets=16, landmarks=16, iters=20)
    dist, st, it = lcn.batched_lcn(ctx, b)
    for k in range(b.count):
        rd, rs = reference(ref, b, k)
        assert st[k] == rs, (k, st[k], rs)
        if rs == 0:
            assert abs(dist[k] - rd) <= 1e-9 * abs(rd), (k, dist[k], rd)
