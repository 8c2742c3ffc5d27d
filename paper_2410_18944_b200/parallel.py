"""Multi-GPU data parallelism over evaluation points (one process per GPU).

Partitioning: rank r owns the contiguous block
[r * N / G, (r + 1) * N / G) of the flattened, row-major evaluation points.
Walk streams are keyed by the GLOBAL point index (Rng::for_walk,
proj/include/wost/rng.hpp:28-32), so uniform-mode results are identical for
any G. The scene / BVH and the guiding field are replicated; each training
minibatch's gradient SUM and record count are allreduced with NCCL over
NVLink inside the library (wostgpu_solver_attach_comm), so every rank applies
the identical Adam step and the fields stay bitwise equal.

Training semantics are global, as in the reference's one-process Engine
(proj/src/guide_train.cpp:111-116, 128): before a round's selection the
ranks' usable-record counts are summed, so the 32,768-record cap and the
16,384-record minibatch apply to the union of the ranks' records. Record
selection keys depend only on (seed, round, global point, depth), so the
union of the per-rank selections IS the single-GPU selection.

`run_host_collective` is the same Engine loop over the library's split-phase
training API with the two reductions done by any torch.distributed backend
(gloo, MPI, ...) instead of the in-library NCCL allreduces.
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


def run_host_collective(solver, dist, seed: int, wpp: int, train_until: int, train_cfg):
    """Engine::run_batch (proj/src/solver.cpp:92-104) over point shards with
    host-side collectives: per training round, collect records, allreduce the
    usable count, select, and per minibatch allreduce the gradient sum (+ its
    record count) and take the Adam step; the frozen-field rounds after
    training run as one multi-round launch. Returns the number of Adam steps."""
    import torch
    steps = 0
    b = 0
    while b < min(wpp, train_until):
        solver.solve_rounds(seed, b, 1, collect=True)
        u = torch.tensor([solver.train_prepare(train_cfg)], dtype=torch.int64)
        dist.all_reduce(u)
        n_mb = solver.train_select(train_cfg, int(u.item()))
        for mb in range(n_mb):
            g = torch.from_numpy(solver.train_minibatch_grad(train_cfg, mb))
            dist.all_reduce(g)
            if g[-1].item() > 0:
                steps += 1
            solver.train_apply(train_cfg, g.numpy())
        b += 1
    if b < wpp:
        solver.solve_rounds(seed, b, wpp - b)
    return steps
