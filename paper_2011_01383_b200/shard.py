"""Multi-GPU sharding of independent structures.

Structures of a batch share nothing (property P.3), so a
batch shards by whole structures: rank r of G takes a contiguous block of
structures, rebases their node ids to 0 and runs cx_linearize + cx_forward on
its own GPU. No data-path collective is needed; the only optional collective
is an all-gather of the packed root states (NCCL over NVLink/NVSwitch, or gloo
on CPU for the tests). This module is host-side index arithmetic only.
"""
from __future__ import annotations

import numpy as np


def block_range(num_structures: int, rank: int, world: int):
    """Contiguous block [g0, g1) of structures owned by `rank` (sizes differ by
    at most one)."""
    q, r = divmod(num_structures, world)
    g0 = rank * q + min(rank, r)
    return g0, g0 + q + (1 if rank < r else 0)


def shard(children: np.ndarray, offsets: np.ndarray, rank: int, world: int, words=None):
    """Rank-local slice of a batch whose structure g occupies input ids
    [offsets[g], offsets[g+1]) (the layout the generators emit).

    Returns (children_local [maxc, n_local] int32, words_local or None,
    (g0, g1), node_offset)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    g0, g1 = block_range(len(offsets) - 1, rank, world)
    a, b = int(offsets[g0]), int(offsets[g1])
    sub = np.array(children[:, a:b], dtype=np.int32, copy=True)
    if sub.size:
        outside = (sub >= 0) & ((sub < a) | (sub >= b))
        if outside.any():
            raise ValueError("a structure references nodes outside its id range")
        sub[sub >= 0] -= a
    w = None if words is None else np.array(words[a:b], copy=True)
    return sub, w, (g0, g1), a


def all_gather_roots(local_roots, num_structures: int, group=None):
    """All-gather the packed root states [local structures, H] of every rank
    into [num_structures, H] (torch.distributed; NCCL on GPUs, gloo on CPU).
    Ranks may own different numbers of structures (padded exchange)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    H = local_roots.shape[1]
    sizes = [block_range(num_structures, r, world) for r in range(world)]
    cap = max(g1 - g0 for g0, g1 in sizes)
    pad = torch.zeros((cap, H), dtype=local_roots.dtype, device=local_roots.device)
    pad[: local_roots.shape[0]] = local_roots
    out = torch.empty((world * cap, H), dtype=local_roots.dtype, device=local_roots.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * cap: r * cap + (g1 - g0)] for r, (g0, g1) in enumerate(sizes)]
    return torch.cat(parts, dim=0)
