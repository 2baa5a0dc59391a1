"""Host logic of the multi-GPU path, mirrored from the
sharded solve in csrc/sinkhorn.cu (Solver::owned_buckets, the row slices and
lcn_iteration_sharded) so it can be tested with gloo on CPU.

One problem over `world` ranks; every rank holds the operator and the full
scaling vectors.
  * Band work: per band and pass, whole buckets go to ranks by
    longest-processing-time greedy on their streamed bytes (`bucket_owners`).
    A rank writes the corrections of its buckets' outputs, zeros elsewhere.
  * Low-rank rows: equal slices of cs = round_up(ceil(n / world), 16) rows
    (`row_slices`).
  * Per half-iteration: reduce-scatter of the per-band corrections onto the
    slices, low-rank pass over the own slice, all-gather of the new log
    vector, and the cross-rank low-rank combine
        H = max_r h_r,   mid = sum_r exp(h_r - H) part_r
    (all-reduce MAX + rescale + all-reduce SUM, `allreduce_lowrank`), plus an
    all-reduce SUM of the marginal-error partial and the error-flag counts.
"""
from __future__ import annotations

import heapq
import math

import numpy as np


def plan_shards(src_counts, tgt_counts, l: int, world: int) -> np.ndarray:
    """Assign buckets to ranks (longest-processing-time greedy, ties to the
    lowest rank). Returns rank per bucket."""
    src = np.asarray(src_counts, dtype=np.int64)
    tgt = np.asarray(tgt_counts, dtype=np.int64)
    if src.shape != tgt.shape:
        raise ValueError("plan_shards: bucket count mismatch")
    cost = src * tgt + (src + tgt) * int(l)
    order = sorted(range(len(cost)), key=lambda b: (-int(cost[b]), b))
    heap = [(0, r) for r in range(world)]
    owner = np.zeros(len(cost), dtype=np.int32)
    for b in order:
        load, r = heapq.heappop(heap)
        owner[b] = r
        heapq.heappush(heap, (load + int(cost[b]), r))
    return owner


def shard_loads(src_counts, tgt_counts, l: int, owner, world: int) -> np.ndarray:
    src = np.asarray(src_counts, dtype=np.int64)
    tgt = np.asarray(tgt_counts, dtype=np.int64)
    cost = src * tgt + (src + tgt) * int(l)
    return np.bincount(np.asarray(owner), weights=cost, minlength=world)


def combine_partials(hs, parts):
    """H = max h_r, mid = sum_r exp(h_r - H) part_r (ranks with h = -inf hold
    no rows)."""
    hs = np.asarray(hs, dtype=np.float64)
    parts = np.asarray(parts, dtype=np.float64)
    H = float(np.max(hs))
    if H == -math.inf:
        return H, np.zeros(parts.shape[1:])
    w = np.where(np.isneginf(hs), 0.0, np.exp(hs - H))
    return H, np.tensordot(w, parts, axes=1)


def allreduce_lowrank(h: float, part, group=None):
    """The per-half-iteration exchange across ranks (torch.distributed; NCCL on
    GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(part, dtype=torch.float64).clone()
    hh = torch.tensor([h], dtype=torch.float64, device=t.device)
    dist.all_reduce(hh, op=dist.ReduceOp.MAX, group=group)
    H = float(hh.item())
    scale = 0.0 if (h == -math.inf or H == -math.inf) else math.exp(h - H)
    t.mul_(scale)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return H, t.cpu().numpy()


def max_over_ranks(x: float, group=None) -> float:
    """Timing rule: report the max over ranks."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def bucket_owners(costs, world: int) -> np.ndarray:
    """Rank per bucket, as Solver::owned_buckets: buckets by decreasing cost
    (stable), each to the least-loaded rank (ties to the lowest rank)."""
    costs = np.asarray(costs, dtype=np.float64)
    order = sorted(range(len(costs)), key=lambda b: -costs[b])  # stable
    heap = [(0.0, r) for r in range(world)]
    owner = np.zeros(len(costs), dtype=np.int32)
    for b in order:
        load, r = heapq.heappop(heap)
        owner[b] = r
        heapq.heappush(heap, (load + float(costs[b]), r))
    return owner


def row_slices(n: int, world: int, align: int = 16):
    """Equal padded slices of the low-rank rows: (cs, [(lo_r, hi_r)])."""
    cs = (-(-n // world) + align - 1) // align * align
    out = []
    for r in range(world):
        lo = min(n, r * cs)
        out.append((lo, min(n, lo + cs)))
    return cs, out
