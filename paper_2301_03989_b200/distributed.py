"""Multi-GPU plumbing for the batch propagator: one process per GPU.

Trajectories shard naturally (independent groups): each rank
propagates a contiguous, group-aligned shard with its own device context; there
is no collective inside the iteration or segment loop.  The only exchange is one
gather of the terminal states at the end (NCCL over NVLink on GPUs; gloo in the
CPU tests), padded to the largest shard because NCCL all-gather needs equal
counts.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_groups(group_sizes: Sequence[int], world: int) -> List[Tuple[int, int, int, int]]:
    """Contiguous group-aligned shards balanced by trajectory count.

    Returns per rank (group_lo, group_hi, traj_lo, traj_hi).  A group never spans
    ranks (block.hpp:83-106 groups are the unit of convergence); rank r takes the
    groups whose first trajectory falls in [r*M/world, (r+1)*M/world).
    """
    sizes = np.asarray(group_sizes, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    total = int(offsets[-1])
    out = []
    g = 0
    for r in range(world):
        hi_traj = (r + 1) * total // world
        g_lo = g
        while g < len(sizes) and offsets[g] < hi_traj:
            g += 1
        if r == world - 1:
            g = len(sizes)
        out.append((g_lo, g, int(offsets[g_lo]), int(offsets[g])))
    return out


def gather_terminal(local: np.ndarray, shards, rank: int, world: int, device=None) -> np.ndarray | None:
    """All-gather the per-rank terminal states [m_r, 7] into the batch order [M, 7].

    Uses torch.distributed (the caller has initialised the process group: NCCL for
    CUDA tensors, gloo for CPU).  Returns the full array on every rank.
    """
    import torch
    import torch.distributed as dist

    counts = [hi - lo for (_, _, lo, hi) in shards]
    pad = max(counts) if counts else 0
    buf = torch.zeros((pad, 7), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    out = torch.empty((world * pad, 7), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, buf)
    host = out.cpu().numpy()
    parts = [host[r * pad: r * pad + counts[r]] for r in range(world)]
    return np.concatenate(parts, axis=0) if parts else np.zeros((0, 7))
