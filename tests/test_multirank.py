"""Multi-rank host logic on CPU: world_size 2 over torch.distributed gloo.

The GPU data path (NCCL allreduce inside the library) cannot run here; these
tests pin the protocol it implements with the CPU oracle:
  * point sharding with global RNG keys reproduces the single-rank run,
  * summing per-rank minibatch gradient SUMS and record counts (what the
    library allreduces) equals the single-rank minibatch mean gradient,
  * per-rank PointStats gathered in rank order equal the single-rank stats.
"""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.parallel import gather_stats, shard_bounds, shard_points
from paper_2410_18944_b200.scene import cell_centers, make_preset


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    from oracle_lib import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("orc")
    pr = make_preset("neumann-strip-vlin")
    h = orc.scene(pr.scene)
    pts = cell_centers(16, 16, pr.eval_bbox)
    mine, off = shard_points(pts, world, rank)
    # uniform walks keyed by global index, 4 wpp rounds, Welford in wpp order
    st = np.zeros(len(mine), dtype=abi.POINT_STATS_DTYPE)
    cfg = abi.solver_config("uniform")
    for w in range(4):
        est, esc, _ = orc.walks(h, None, cfg, mine, 3, w, point_index=np.arange(off, off + len(mine)))
        for i, v in enumerate(est):
            c = st[i]["count"] + 1
            d = v - st[i]["mean"]
            st[i]["count"] = c
            st[i]["mean"] += d / c
            st[i]["m2"] += d * (v - st[i]["mean"])
    full = gather_stats(dist, st, world)
    # gradient protocol: sum of per-rank sums / global count == global mean
    f = orc.field(abi.field_config(), pr.scene.bbox, 9)
    sol_st = np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE)
    recs = orc.solve_batch(h, f, abi.solver_config("learnable_mis"), pts, sol_st, 4, 0, collect=True)
    recs = recs[:2000]
    b, e = shard_bounds(len(recs), world, rank)
    tc = abi.train_config()
    g_sum = torch.tensor(orc.field_grad(f, recs[b:e], tc) * (e - b), dtype=torch.float64)
    cnt = torch.tensor([float(e - b)], dtype=torch.float64)
    dist.all_reduce(g_sum)
    dist.all_reduce(cnt)
    if rank == 0:
        out["stats"] = full
        out["grad"] = (g_sum / cnt).numpy()
    dist.destroy_process_group()


def test_two_rank_protocol_matches_single_rank(orc):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    pr = make_preset("neumann-strip-vlin")
    h = orc.scene(pr.scene)
    pts = cell_centers(16, 16, pr.eval_bbox)
    st = np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE)
    for w in range(4):
        orc.solve_batch(h, None, abi.solver_config("uniform"), pts, st, 3, w)
    full = out["stats"]
    assert np.array_equal(full["count"], st["count"])
    np.testing.assert_allclose(full["mean"], st["mean"], rtol=0, atol=1e-15)
    f = orc.field(abi.field_config(), pr.scene.bbox, 9)
    sol_st = np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE)
    recs = orc.solve_batch(h, f, abi.solver_config("learnable_mis"), pts, sol_st, 4, 0, collect=True)
    g = orc.field_grad(f, recs[:2000], abi.train_config())
    np.testing.assert_allclose(out["grad"], g, rtol=1e-9, atol=1e-15)


def _worker3(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import Oracle3
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o3 = Oracle3()
    h = o3.scene(make_preset3("box-strip-vlin", n=6).scene)
    pts = slice_points(12, 12)
    mine, off = shard_points(pts, world, rank)
    # 3D walks keyed by the GLOBAL point index (cfg 5 sharding)
    st = o3.run(h, None, abi.solver_config("uniform"), mine, 5, 3, point_offset=off)
    full = gather_stats(dist, st, world)
    if rank == 0:
        out["stats"] = full
    dist.destroy_process_group()


def test_two_rank_3d_sharding_matches_single_rank():
    """cfg 5's protocol on the 3D oracle: points sharded over ranks with walk
    streams keyed by the global index give the single-rank statistics."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import Oracle3
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker3, args=(2, _port(), out), nprocs=2, join=True)
    o3 = Oracle3()
    h = o3.scene(make_preset3("box-strip-vlin", n=6).scene)
    st = o3.run(h, None, abi.solver_config("uniform"), slice_points(12, 12), 5, 3)
    full = out["stats"]
    assert np.array_equal(full["count"], st["count"])
    assert np.array_equal(full["mean"], st["mean"])


def test_shard_bounds_cover_all_points():
    for n in (1, 7, 16384, 16385):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
