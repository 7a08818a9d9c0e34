"""Multi-GPU plumbing for the batch propagator: one process per GPU.

Trajectories shard naturally (independent groups): each rank
propagates a contiguous, group-aligned shard with its own device context; there
is no collective inside the iteration or segment loop.  The only exchange is one
gather of the terminal states to rank 0 at the end (NCCL over NVLink on GPUs;
gloo in the CPU tests), padded to the largest shard.
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


def gather_terminal(local: np.ndarray, shards, rank: int, world: int, device=None, dst: int = 0) -> np.ndarray | None:
    """Gather the per-rank terminal states [m_r, 7] to rank `dst` in batch order [M, 7].

    One collective (torch.distributed.gather: NCCL send/recv over NVLink for CUDA tensors,
    gloo for CPU tensors) of buffers padded to the largest shard.  Returns the full array
    on `dst` and None elsewhere (only the destination copies to the host).
    """
    import torch
    import torch.distributed as dist

    counts = [hi - lo for (_, _, lo, hi) in shards]
    pad = max(counts) if counts else 0
    buf = torch.zeros((pad, 7), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst)
    if rank != dst:
        return None
    host = torch.cat(parts).cpu().numpy()
    return np.concatenate([host[r * pad: r * pad + counts[r]] for r in range(world)], axis=0)
