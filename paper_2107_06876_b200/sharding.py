"""Host logic of the multi-GPU path.

Points are sharded across GPUs by round-1 LSH bucket so that every band-0
K_sp / K_Delta block stays on one GPU; whole buckets are assigned greedily to
balance  sum_b n_b m_b + (n_b + m_b) l  (block entries + low-rank rows).
The only exchange per half-iteration is the low-rank partial: each rank holds
(h_r, part_r = sum_{own rows} F_row exp(v_row - h_r)), and
    H = max_r h_r,   mid = sum_r exp(h_r - H) part_r,
which is exactly the cross-block combine of lowrank_reduce_kernel
(csrc/sinkhorn.cu) lifted to ranks: one all-reduce(MAX) of h and one
all-reduce(SUM) of l values (+ the marginal-error scalar) per half-iteration.
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
