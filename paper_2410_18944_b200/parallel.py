"""Multi-GPU data parallelism over evaluation points (one process per GPU).

Partitioning: rank r owns the contiguous block
[r * N / G, (r + 1) * N / G) of the flattened, row-major evaluation points.
Walk streams are keyed by the GLOBAL point index (Rng::for_walk,
proj/include/wost/rng.hpp:28-32), so uniform-mode results are identical for
any G. The scene / BVH and the guiding field are replicated; each training
minibatch's gradient SUM and record count are allreduced with NCCL over
NVLink inside the library (wostgpu_solver_attach_comm), so every rank applies
the identical Adam step and the fields stay bitwise equal.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n_points: int, world: int, rank: int):
    """[begin, end) of rank's contiguous block of the global point list."""
    base, rem = divmod(n_points, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def shard_points(points: np.ndarray, world: int, rank: int):
    """Rank's points and the global index of its first point."""
    b, e = shard_bounds(len(points), world, rank)
    return np.ascontiguousarray(points[b:e]), b


def broadcast_comm_id(dist, rank: int):
    """Rank 0 creates the NCCL unique id (128 bytes) and broadcasts it over
    torch.distributed (any backend)."""
    obj = [None]
    if rank == 0:
        from .api import comm_unique_id
        obj[0] = comm_unique_id()
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def gather_stats(dist, stats: np.ndarray, world: int):
    """Concatenate every rank's PointStats block on all ranks (global order)."""
    parts = [None] * world
    dist.all_gather_object(parts, stats)
    return np.concatenate(parts)
