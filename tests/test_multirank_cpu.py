"""Multi-rank host logic on CPU (gloo, world_size 2): the per-half-iteration
low-rank exchange of the sharded solve and the max-over-ranks timing rule
(SURVEY.md §8(e)), plus the bucket-to-rank planner."""
import math
import os
import socket

import numpy as np
import pytest

from paper_2107_06876_b200 import sharding


def test_plan_shards_balances_and_is_deterministic():
    r = np.random.default_rng(3)
    src = r.integers(0, 600, 4096)
    tgt = r.integers(0, 600, 4096)
    own = sharding.plan_shards(src, tgt, 512, 8)
    assert np.array_equal(own, sharding.plan_shards(src, tgt, 512, 8))
    loads = sharding.shard_loads(src, tgt, 512, own, 8)
    assert loads.max() / loads.mean() < 1.01
    assert set(own.tolist()) == set(range(8))


def test_combine_partials_matches_global_shift():
    r = np.random.default_rng(5)
    v = r.normal(0, 30, 1000)            # log scalings
    F = r.uniform(0, 1, (1000, 16))      # factor rows
    want = F.T @ np.exp(v - v.max())
    chunks = np.array_split(np.arange(1000), 7)
    hs, parts = [], []
    for c in chunks:
        h = v[c].max()
        hs.append(h)
        parts.append(F[c].T @ np.exp(v[c] - h))
    hs.append(-math.inf)                 # an empty rank
    parts.append(np.zeros(16))
    H, mid = sharding.combine_partials(hs, parts)
    assert H == v.max()
    assert np.allclose(mid, want, rtol=1e-13)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = np.random.default_rng(100 + rank)
    h = float(r.normal(0, 40))
    part = r.uniform(0, 1, 8)
    H, mid = sharding.allreduce_lowrank(h, part)
    t = sharding.max_over_ranks(float(rank) + 0.5)
    q.put((rank, h, part, H, mid, t))
    dist.destroy_process_group()


def test_gloo_allreduce_lowrank_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    out.sort(key=lambda x: x[0])
    hs = [o[1] for o in out]
    parts = [o[2] for o in out]
    H, mid = sharding.combine_partials(hs, parts)
    for o in out:
        assert o[3] == H
        assert np.allclose(o[4], mid, rtol=1e-14)
        assert o[5] == 1.5


def test_bucket_owners_and_row_slices_partition():
    r = np.random.default_rng(7)
    costs = r.uniform(1, 1e4, 500)
    for world in (1, 2, 3, 8):
        own = sharding.bucket_owners(costs, world)
        assert set(own.tolist()) <= set(range(world))
        loads = np.bincount(own, weights=costs, minlength=world)
        assert loads.max() - loads.min() <= costs.max()  # LPT bound
        cs, sl = sharding.row_slices(1000, world)
        assert cs % 16 == 0 and cs * world >= 1000
        covered = np.concatenate([np.arange(lo, hi) for lo, hi in sl])
        assert np.array_equal(covered, np.arange(1000))


def _half_iteration(rank, world, data, comm):
    """One row half-iteration of the sharded solve, numpy per rank +
    collectives through `comm` (None = single rank)."""
    U, mid_parts, corr_blocks, log_marg, owners = data
    n, l = U.shape
    # band corrections: own buckets only, zeros elsewhere (then the exchange)
    corr = np.zeros(n)
    for b, (rows, vals) in enumerate(corr_blocks):
        if comm is None or owners[b] == rank:  # single rank: every bucket
            corr[rows] = vals
    if comm:
        corr = comm["allreduce_sum"](corr)  # reduce-scatter, read back as the full vector
    cs, sl = sharding.row_slices(n, world)
    lo, hi = sl[rank]
    # cross-rank combine of the previous half's low-rank partials
    h_r, part_r = mid_parts[rank] if comm else sharding.combine_partials(*zip(*mid_parts))
    H, mid = comm["lowrank"](h_r, part_r) if comm else (h_r, part_r)
    y = U[lo:hi] @ (mid * np.exp(H)) + corr[lo:hi]
    log_out = np.full(n, np.nan)
    log_out[lo:hi] = log_marg[lo:hi] - np.log(y)
    if comm:
        log_out = comm["allgather"](log_out[lo:hi], cs, n)
    # this rank's partial for the next half (own rows, own shift)
    v = log_out[lo:hi]
    h = float(v.max()) if hi > lo else -math.inf
    part = U[lo:hi].T @ np.exp(v - h) if hi > lo else np.zeros(l)
    if comm:
        h, part = comm["lowrank"](h, part)
    else:
        h, part = h, part
    return log_out, h, part


def _sharded_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    data = _sharded_problem(world)

    def allreduce_sum(x):
        t = torch.from_numpy(x.copy())
        dist.all_reduce(t)
        return t.numpy()

    def allgather(own, cs, n):
        buf = torch.zeros(cs, dtype=torch.float64)
        buf[:len(own)] = torch.from_numpy(own)
        outs = [torch.zeros(cs, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(outs, buf)
        return torch.cat(outs).numpy()[:n]

    comm = {"allreduce_sum": allreduce_sum, "allgather": allgather, "lowrank": sharding.allreduce_lowrank}
    q.put((rank,) + _half_iteration(rank, world, data, comm))
    dist.destroy_process_group()


def _sharded_problem(world):
    r = np.random.default_rng(11)
    n, l, nbk = 200, 12, 17
    U = r.uniform(0.1, 1.0, (n, l))
    bucket = r.integers(0, nbk, n)
    corr_blocks = [(np.flatnonzero(bucket == b), r.uniform(-0.05, 0.05, int((bucket == b).sum()))) for b in range(nbk)]
    costs = [len(rows) for rows, _ in corr_blocks]
    owners = sharding.bucket_owners(costs, world)
    log_marg = np.log(np.full(n, 1.0 / n))
    # previous half's partials: rank slices of a common vector
    v = r.normal(0, 3, n)
    cs, sl = sharding.row_slices(n, world)
    mid_parts = []
    for lo, hi in sl:
        h = float(v[lo:hi].max())
        mid_parts.append((h, U[lo:hi].T @ np.exp(v[lo:hi] - h)))
    return U, mid_parts, corr_blocks, log_marg, owners


def test_gloo_sharded_half_iteration_matches_single_rank():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    # single-rank reference of the same half-iteration
    data = _sharded_problem(world)
    ref_log, ref_h, ref_part = _half_iteration(0, 1, data, None)
    for _, log_out, h, part in out:
        assert np.allclose(log_out, ref_log, rtol=1e-13, atol=0)
        H, mid = sharding.combine_partials([ref_h], [ref_part])
        assert h == H
        assert np.allclose(part, mid, rtol=1e-12)
