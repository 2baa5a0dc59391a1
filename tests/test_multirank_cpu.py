"""Multi-rank logic of the bucket-sharded solve on CPU.

The partition comes from the library itself (lcn_shard_plan_*, host-only
C-ABI of liblcn_b200.so, no GPU needed): the same code the sharded build
runs. The tests check the plan's invariants (owned points partition the
problem, every support pair of an owned point is local, the exchange maps
point at the right values) and run the sharded LCN-Sinkhorn data flow in
numpy over gloo, world_size 2 and 3: each rank holds only its local block
of the support and its factor rows; per half-iteration ONE all-gather of
[shift | low-rank partial | exported scalings] -- the record the CUDA path
all-gathers (sinkhorn.cu lcn_iteration_shard); the gathered result equals the
single-rank solve."""
import math
import os
import socket

import numpy as np
import pytest

from paper_2107_06876_b200.native import ShardPlan


def _ids(seed, n, m, bands, buckets, coherent):
    """Bucket ids per band. coherent: later bands re-cluster band 0 (k-means
    LSH on clustered data: most later buckets sit inside one band-0 group);
    otherwise independent random buckets (large halos)."""
    r = np.random.default_rng(seed)
    src = np.zeros((bands, n), np.uint32)
    tgt = np.zeros((bands, m), np.uint32)
    src[0] = r.integers(0, buckets, n)
    tgt[0] = r.integers(0, buckets, m)
    for b in range(1, bands):
        if coherent:
            perm = r.permutation(buckets)
            flip_s = r.random(n) < 0.05
            flip_t = r.random(m) < 0.05
            src[b] = np.where(flip_s, r.integers(0, buckets, n), perm[src[0]])
            tgt[b] = np.where(flip_t, r.integers(0, buckets, m), perm[tgt[0]])
        else:
            src[b] = r.integers(0, buckets, n)
            tgt[b] = r.integers(0, buckets, m)
    return src, tgt


def _support(src, tgt):
    """Dense mask of the union of the bands' bucket blocks (lsh.cpp:212-243)."""
    return (src[:, :, None] == tgt[:, None, :]).any(axis=0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("coherent", [True, False])
def test_shard_plan_invariants(world, coherent):
    n, m, bands, buckets = 300, 260, 2, 24
    src, tgt = _ids(5 + world, n, m, bands, buckets, coherent)
    plan = ShardPlan(src, tgt, buckets, 16, world)
    sup = _support(src, tgt)
    own_s, own_t = np.full(n, -1), np.full(m, -1)
    infos, pts, exch = [], [], []
    for r in range(world):
        i = plan.info(r)
        s_loc, t_loc = plan.points(r)
        infos.append(i)
        pts.append((s_loc, t_loc))
        exch.append(plan.exchange(r))
        assert len(s_loc) == i["n_own"] + i["n_halo"] and len(t_loc) == i["m_own"] + i["m_halo"]
        # owned ascending then halo ascending, no repeats
        for loc, no in ((s_loc, i["n_own"]), (t_loc, i["m_own"])):
            assert np.all(np.diff(loc[:no].astype(np.int64)) > 0)
            assert np.all(np.diff(loc[no:].astype(np.int64)) > 0)
            assert len(np.intersect1d(loc[:no], loc[no:])) == 0
        assert np.all(own_s[s_loc[:i["n_own"]]] == -1) and np.all(own_t[t_loc[:i["m_own"]]] == -1)
        own_s[s_loc[:i["n_own"]]] = r
        own_t[t_loc[:i["m_own"]]] = r
    assert np.all(own_s >= 0) and np.all(own_t >= 0)          # the owned points partition the problem
    # band-0 buckets are the shard unit: both sides of a bucket on one rank
    for c in range(buckets):
        ranks = set(own_s[src[0] == c].tolist()) | set(own_t[tgt[0] == c].tolist())
        assert len(ranks) <= 1
    # every support pair of an owned point is local to its rank
    for r in range(world):
        s_loc, t_loc = pts[r]
        ls, lt = np.zeros(n, bool), np.zeros(m, bool)
        ls[s_loc] = True
        lt[t_loc] = True
        rows = own_s == r
        cols = own_t == r
        assert not np.any(sup[rows][:, ~lt]), "an owned source has a support target outside the rank"
        assert not np.any(sup[:, cols][~ls, :]), "an owned target has a support source outside the rank"
        # halo points are needed: each shares a later-band bucket with an owned point of the other side
        nh = infos[r]["n_own"]
        for g in s_loc[nh:]:
            assert np.any(sup[g, cols])
    # exchange maps: halo value k of rank r is slot imp_slot[k] of rank imp_rank[k]'s export
    for r in range(world):
        s_loc, t_loc = pts[r]
        for side, loc, no in (("s", s_loc, infos[r]["n_own"]), ("t", t_loc, infos[r]["m_own"])):
            e = exch[r]
            for k, g in enumerate(loc[no:]):
                o, slot = e[f"imp_{side}_rank"][k], e[f"imp_{side}_slot"][k]
                o_loc = pts[o][0 if side == "s" else 1]
                assert o_loc[exch[o][f"exp_{side}"][slot]] == g
            assert len(e[f"exp_{side}"]) <= infos[r][f"max_exp_{side}"]
    if world == 1:
        assert infos[0]["n_halo"] == 0 and infos[0]["m_halo"] == 0
    # deterministic: every rank computes the same plan
    again = ShardPlan(src, tgt, buckets, 16, world)
    for r in range(world):
        a, b = again.points(r), pts[r]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_shard_plan_groups_band0_buckets_a_later_band_joins():
    """k-means LSH bands on clustered data re-cluster the same groups
    (configs[3]: 1000 mixture components, both bands' 4096 buckets nest in
    them; the plan there has no halo at all, profiles/shard_plan_c3.json).
    Here band 1 joins band-0 buckets in threes: the affinity grouping keeps
    each joined triple on one rank, so nothing is exchanged, and the load
    stays balanced."""
    r = np.random.default_rng(2)
    n = m = 6000
    buckets = 96
    src0 = r.integers(0, buckets, n).astype(np.uint32)
    tgt0 = r.integers(0, buckets, m).astype(np.uint32)
    perm = r.permutation(buckets)
    src = np.stack([src0, (perm[src0] // 3).astype(np.uint32)])
    tgt = np.stack([tgt0, (perm[tgt0] // 3).astype(np.uint32)])
    for world in (2, 4, 8):
        plan = ShardPlan(src, tgt, buckets, 32, world)
        infos = [plan.info(k) for k in range(world)]
        assert sum(i["n_halo"] + i["m_halo"] for i in infos) == 0
        assert infos[0]["max_exp_s"] == 0 and infos[0]["max_exp_t"] == 0
        own = np.array([i["n_own"] + i["m_own"] for i in infos])
        assert own.max() < 1.25 * own.mean()


def test_shard_plan_rejects_bad_input():
    from paper_2107_06876_b200 import InvalidArgument
    src = np.zeros((1, 10), np.uint32)
    tgt = np.zeros((1, 10), np.uint32)
    with pytest.raises(InvalidArgument, match="world size"):
        ShardPlan(src, tgt, 4, 8, 0)
    with pytest.raises(InvalidArgument, match="out of range"):
        ShardPlan(src + 7, tgt, 4, 8, 2)


# ---------------------------------------------------------------------------
# sharded LCN-Sinkhorn data flow over gloo
# ---------------------------------------------------------------------------
def _problem(seed=3):
    r = np.random.default_rng(seed)
    n, m, d, l, buckets = 160, 140, 3, 6, 12
    p = r.normal(size=(n, d))
    q = r.normal(size=(m, d)) * 1.1
    src, tgt = _ids(seed, n, m, 2, buckets, False)
    lam = 2.0
    C = ((p[:, None, :] - q[None, :, :]) ** 2).sum(-1)
    L = np.concatenate([p[:l // 2], q[:l - l // 2]])
    U = np.exp(-((p[:, None, :] - L[None]) ** 2).sum(-1) / lam)
    A = np.exp(-((L[:, None, :] - L[None]) ** 2).sum(-1) / lam)
    V = np.exp(-((L[:, None, :] - q[None]) ** 2).sum(-1) / lam)
    W = np.linalg.solve(A + 1e-9 * np.eye(l), V)               # K_nys = U W (l x m)
    sup = _support(src, tgt)
    delta = np.where(sup, np.exp(-C / lam) - U @ W, 0.0)        # LCN correction on the support
    a = np.full(n, 1.0 / n)
    b = np.full(m, 1.0 / m)
    return dict(src=src, tgt=tgt, buckets=buckets, U=U, W=W, delta=delta, a=a, b=b, l=l)


ITERS = 25


def _single(pb):
    """Unsharded reference: t-half then s-half, as the device loop."""
    K = pb["U"] @ pb["W"] + pb["delta"]
    s = np.ones(len(pb["a"]))
    for _ in range(ITERS):
        t = pb["b"] / (K.T @ s)
        s = pb["a"] / (K @ t)
    return s, t


def _sharded(rank, world, pb, allgather):
    """This rank's half of the data flow: local block of delta (owned + halo
    points, built from the bucket ids the way the library builds it: halo
    band-0 ids relabelled one-sided), factor rows of the local points, one
    all-gather per half-iteration."""
    plan = ShardPlan(pb["src"], pb["tgt"], pb["buckets"], pb["l"], world)
    info = plan.info(rank)
    s_loc, t_loc = plan.points(rank)
    ex = plan.exchange(rank)
    ns, mt = info["n_own"], info["m_own"]
    src = pb["src"][:, s_loc].copy()
    tgt = pb["tgt"][:, t_loc].copy()
    src[0, ns:] = pb["buckets"]          # halo sources: a one-sided band-0 bucket
    tgt[0, mt:] = pb["buckets"] + 1      # halo targets: another one
    local_sup = _support(src, tgt)
    D = np.where(local_sup, pb["delta"][np.ix_(s_loc, t_loc)], 0.0)
    U, Wt = pb["U"][s_loc], pb["W"][:, t_loc].T
    a, b = pb["a"][s_loc], pb["b"][t_loc]
    l = pb["l"]
    X_s, X_t = info["max_exp_s"], info["max_exp_t"]
    s = np.ones(len(s_loc))
    t = np.zeros(len(t_loc))

    def exchange(vec, own, partial_rows, F, exp_idx, X, imp_rank, imp_slot):
        # record: [partial (l) | exported values padded to X]
        rec = np.zeros(l + X)
        rec[:l] = F[:own].T @ partial_rows
        rec[l:l + len(exp_idx)] = vec[exp_idx]
        allr = allgather(rec)                                     # world x (l + X)
        mid = allr[:, :l].sum(axis=0)                              # rank order
        vec[own:] = allr[imp_rank, l + imp_slot]
        return mid

    mid_s = exchange(s, ns, s[:ns], U, ex["exp_s"], X_s, ex["imp_s_rank"], ex["imp_s_slot"])  # U^T s, s = 1
    for _ in range(ITERS):
        t[:mt] = b[:mt] / (Wt[:mt] @ mid_s + D[:, :mt].T @ s)
        mid_t = exchange(t, mt, t[:mt], Wt, ex["exp_t"], X_t, ex["imp_t_rank"], ex["imp_t_slot"])
        s[:ns] = a[:ns] / (U[:ns] @ mid_t + D[:ns] @ t)
        mid_s = exchange(s, ns, s[:ns], U, ex["exp_s"], X_s, ex["imp_s_rank"], ex["imp_s_slot"])
    return s_loc[:ns], s[:ns], t_loc[:mt], t[:mt], info


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allgather(rec):
            x = torch.from_numpy(rec.copy())
            outs = [torch.zeros_like(x) for _ in range(world)]
            dist.all_gather(outs, x)
            return torch.stack(outs).numpy()

        q.put((rank,) + _sharded(rank, world, _problem(), allgather))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_solve_matches_single_rank(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    pb = _problem()
    s_ref, t_ref = _single(pb)
    s = np.full(len(s_ref), np.nan)
    t = np.full(len(t_ref), np.nan)
    halo = 0
    for _, gs, vs, gt, vt, info in out:
        s[gs] = vs
        t[gt] = vt
        halo += info["n_halo"] + info["m_halo"]
    assert halo > 0, "the random bands should leave halo points to exchange"
    assert np.allclose(s, s_ref, rtol=1e-12, atol=0)
    assert np.allclose(t, t_ref, rtol=1e-12, atol=0)
