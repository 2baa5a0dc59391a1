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
