"""Config-space sharding and the single collective of the multi-GPU path
(SURVEY.md §8e): configs are dealt to ranks by descending estimated cost
(round robin, so every rank gets a similar mix of heavy and light configs),
each rank evaluates its shard, and one all-gather of the fixed-size
per-config records precedes the global ranking on the device.

Backend-agnostic: NCCL with device tensors in bench.py, gloo with host
tensors in tests/test_dist.py.
"""

from __future__ import annotations

import numpy as np


def config_cost(block_dims: np.ndarray, n_accesses: np.ndarray) -> np.ndarray:
    """Relative cost estimate per config: intervals scale with thread rows
    (threads / BX) times accesses."""
    bd = np.asarray(block_dims, dtype=np.int64).reshape(-1, 3)
    t = bd.prod(axis=1)
    return (t // np.maximum(bd[:, 0], 1) + 1) * np.asarray(n_accesses, dtype=np.int64)


def shard_indices(cost: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Indices of this rank's shard: deal configs sorted by descending cost
    round robin; stable, deterministic, every index on exactly one rank."""
    order = np.argsort(-np.asarray(cost), kind="stable")
    return np.sort(order[rank::world])


# Relative device cost of one configuration's computed work per template
# kind, measured on one B200 (C5 halves evaluated separately, DESIGN.md §5:
# stencil part 311 ms over its sharing groups' config_cost sum 3.4e8, LBM
# part 186 ms over 4.8e7): an LBM unit costs ~4.2x a stencil unit of equal
# config_cost (bitmap-tier key ranges, pattern runs).
KIND_WEIGHT = {"star": 1.0, "jacobi2d": 1.0, "lbm": 4.2}


def group_shards(cost: np.ndarray, group: np.ndarray, world: int) -> list[np.ndarray]:
    """Every rank's shard when configurations that share work (equal
    ``group`` id: exact translates of one another's set problems, see
    csrc/k_dedup.cu) must stay on one rank: the sharing is per rank, so a
    group split over ranks is computed once per rank.  A group costs its
    most expensive member (the others copy); groups are dealt longest
    first to the least-loaded rank (LPT), deterministically.  Returns the
    sorted global indices of each rank."""
    import heapq

    cost = np.asarray(cost, dtype=np.float64)
    gid, inv = np.unique(np.asarray(group), return_inverse=True)
    gcost = np.zeros(len(gid))
    np.maximum.at(gcost, inv, cost)
    order = np.argsort(-gcost, kind="stable")
    owner = np.empty(len(gid), dtype=np.int64)
    heap = [(0.0, r) for r in range(world)]
    for g in order.tolist():
        load, r = heapq.heappop(heap)
        owner[g] = r
        heapq.heappush(heap, (load + float(gcost[g]), r))
    mine = owner[inv]
    return [np.flatnonzero(mine == r) for r in range(world)]


def pad_to(n: int, world: int) -> int:
    """Shard length every rank pads to (all-gather needs equal sizes)."""
    return -(-n // world)


def gather_records(local, world: int, group=None):
    """All-gather a [m][k] records tensor (equal m on every rank of
    ``group``) into [world*m][k] with torch.distributed (one collective)."""
    import torch
    import torch.distributed as dist

    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if hasattr(dist, "all_gather_into_tensor") and local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    else:
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local.contiguous(), group=group)
        out = torch.cat(parts, dim=0)
    return out


def global_index(shards: list[np.ndarray], m: int) -> np.ndarray:
    """Map gathered rows (rank r, slot j) back to global config indices;
    padding slots map to -1."""
    out = np.full(len(shards) * m, -1, dtype=np.int64)
    for r, idx in enumerate(shards):
        out[r * m:r * m + len(idx)] = idx
    return out
