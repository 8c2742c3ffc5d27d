"""Benchmark: guided walk-on-stars walks/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "cfg 2"): preset neumann-strip-vlin
(proj/src/presets.cpp:217-221), 128x128 cell-centre grid per GPU, 256 walks
per point, learnable-MIS guiding with online training in every round
(train_until = 256), default FieldConfig / TrainConfig / SolverConfig, seed 1.
One step = one complete solve of that configuration (256 wpp rounds, each a
device walk round plus a training round) = 4,194,304 walks per GPU.

  python bench.py [--gpus N --steps K --warmup W]          our CUDA path
  python bench.py --impl reference [...]                   the reference C++ on host cores
  python bench.py --workload cfg4|cfg5 [...]               the 3D path (configs[3], configs[4])

N > 1 (torchrun, one rank per GPU): weak scaling; rank r owns rows
[128 r, 128 r + 128) of a 128 x 128N grid over the same domain (global point
index keys every walk's stream), guiding-field gradients are allreduced over
NVLink with NCCL before every Adam step.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PRESET = "neumann-strip-vlin"
GRID = 128
WPP = 256
TRAIN_UNTIL = 256
SEED = 1
# algorithmic HBM bytes per walk step: 52 B SoA walk state read
# + written = 104 B; training rounds add a 56 B trace record written + read
BYTES_PER_STEP = 104
BYTES_PER_TRAIN_STEP = 112


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def flush_l2(buf):
    """Write a buffer larger than the 126 MB L2 between timed steps."""
    if buf is not None:
        buf.zero_()


def cpu_reference_rate(rounds, threads, preset=PRESET, grid=GRID, mode=3):
    """The reference's own run_solve (oracle/_ref, Release-flag build) on the
    host cores for a bounded number of wpp rounds of the same workload."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_FAST_SO, REF_SO, Oracle
    so = REF_FAST_SO if os.path.exists(REF_FAST_SO) else REF_SO
    kind = "reference"
    if not os.path.exists(so):
        return None
    os.environ["OMP_NUM_THREADS"] = str(threads)
    os.environ["WOST_THREADS"] = str(threads)
    ref = Oracle("ref", so)
    sec, rel, tsec = (np.zeros(1) for _ in range(3))
    import ctypes as C
    rc = ref.lib.ref_run_solve(preset.encode(), grid, grid, rounds, mode, TRAIN_UNTIL, SEED, None,
                               sec.ctypes.data_as(C.POINTER(C.c_double)),
                               rel.ctypes.data_as(C.POINTER(C.c_double)),
                               tsec.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        return None
    walks = grid * grid * rounds
    return {"value": walks / float(sec[0]), "seconds": float(sec[0]), "kind": kind,
            "train_seconds": float(tsec[0]), "walks": walks}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rounds = args.ref_rounds
    for _ in range(args.warmup):
        cpu_reference_rate(rounds, threads)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_reference_rate(rounds, threads)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        vals.append(r["value"])
        secs.append(r["seconds"])
    value = float(np.mean(vals))
    sample = (f"{rounds} of {WPP} wpp rounds of cfg 2 ({PRESET} {GRID}x{GRID}, learnable MIS, "
              f"training every round) through the reference's run_solve")
    line = {"metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s",
            "impl": "reference", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(secs)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg2 {PRESET} {GRID}x{GRID} learnable_mis wpp sample {rounds}",
                       "preset": PRESET, "grid": [GRID, GRID], "rounds_per_step": rounds},
            "cpu_baseline": {"value": value, "unit": "walks/s", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "walks/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- 3D (cfg 4 / 5)
# cfg 4 (BASELINE.json configs[3]): box-strip-vlin, the unit box as 99,372
# triangles (Dirichlet x = 0 / x = 1, insulated lateral faces), a 512 x 512
# slice at z = 0.5, 1024 walks per point, learnable MIS with online training
# for the first 256 rounds. cfg 5 (configs[4]): the same domain, 2048 x 2048 =
# 4,194,304 points x 1024 walks sharded over the GPUs (strong scaling).
# Algorithmic HBM bytes per 3D walk step: 60 B SoA state read +
# written = 120 B; training rounds add a 68 B record written + read = 136 B.
BYTES_PER_STEP3 = 120
BYTES_PER_TRAIN_STEP3 = 136


def cpu_oracle3_rate(grid, rounds, train_until, threads):
    """The 3D oracle (oracle/wost3d.inc, a port: the reference has no 3D code)
    on the host cores: `rounds` wpp rounds of the same workload on a grid x
    grid slice."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle3
    from paper_2410_18944_b200 import abi
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points
    os.environ["OMP_NUM_THREADS"] = str(threads)
    o3 = Oracle3()
    p = make_preset3("box-strip-vlin")
    h = o3.scene(p.scene)
    f = o3.field(abi.field_config3(), (0, 0, 0, 1, 1, 1), SEED)
    x = slice_points(grid, grid)
    t0 = time.perf_counter()
    o3.run(h, f, abi.solver_config("learnable_mis"), x, SEED, rounds, train_until, abi.train_config(seed=SEED))
    sec = time.perf_counter() - t0
    o3.field_destroy(f)
    o3.scene_destroy(h)
    walks = grid * grid * rounds
    return {"value": walks / sec, "seconds": sec, "walks": walks, "kind": "port"}


def main3(args):
    cfg5 = args.workload == "cfg5"
    grid = args.grid or (2048 if cfg5 else 512)
    wpp = args.wpp or 1024
    train_until = min(args.train_until, wpp)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # the 3D oracle port on the host cores
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        g, r = 48, 2
        for _ in range(args.warmup):
            cpu_oracle3_rate(g, r, r, threads)
        rr = [cpu_oracle3_rate(g, r, r, threads) for _ in range(args.steps)]
        value = float(np.mean([x["value"] for x in rr]))
        sample = (f"{r} wpp rounds (both training rounds) of a {g}x{g} slice of {args.workload}'s domain "
                  f"through the 3D oracle port (oracle/wost3d.inc; the reference has no 3D code)")
        print(json.dumps({"metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s",
                          "impl": "reference", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": float(np.mean([x["seconds"] for x in rr])) * 1e3,
                          "higher_is_better": True, "scaling": "strong" if cfg5 else "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": f"{args.workload} oracle-port sample {g}x{g} x {r} wpp"},
                          "cpu_baseline": {"value": value, "unit": "walks/s", "cores": threads, "kind": "port",
                                           "sample": sample},
                          "e2e": {"value": value, "unit": "walks/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import torch
    from paper_2410_18944_b200 import _lib, abi
    from paper_2410_18944_b200.api3 import Accel3, GuidingField3, MLP_TENSOR, Solver3
    from paper_2410_18944_b200.parallel import broadcast_comm_id, shard_points
    from paper_2410_18944_b200.scene import relmse
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points, strip_vlin_np

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.init(local)
    preset = make_preset3("box-strip-vlin")
    # cfg 5: strong scaling, the fixed 2048^2 slice split over ranks; cfg 4: weak
    # scaling, rank r owns rows [grid r, grid (r+1)) of a grid x grid*world slice
    all_pts = slice_points(grid, grid if cfg5 else grid * world)
    pts, offset = shard_points(all_pts, world, rank)
    n_local = len(pts)
    box = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    field = GuidingField3(abi.field_config3(), box, SEED)
    p0, m0, v0, s0 = field.state()
    acc = Accel3(preset.scene)
    solver = Solver3(acc, field, abi.solver_config("learnable_mis"), MLP_TENSOR)
    if world > 1:
        solver.attach_comm(broadcast_comm_id(dist, rank), world, rank)
    tcfg = abi.train_config(seed=SEED)
    solver.set_points(pts, offset)
    l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step():
        field.set_state(p0, m0, v0, s0)
        flush_l2(l2)
        torch.cuda.synchronize()
        _, ms = solver.run(SEED, wpp, train_until, tcfg)
        return ms

    for _ in range(args.warmup):
        one_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    times, prof = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            times.append(one_step())
            prof.append(solver.run_profile())
    launches = (_lib.kernel_launches() - launches0) // max(1, args.steps)
    total_ms = float(np.sum(times))
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    walks_per_step = len(all_pts) * wpp
    value = walks_per_step * args.steps / (total_ms * 1e-3)
    ref = strip_vlin_np(pts[:, 0], pts[:, 1])
    rel_guided = relmse(solver.stats()["mean"], ref)
    pr = prof[-1]
    peaks, peak_kind = measured_peaks()
    alg = pr["steps"] * BYTES_PER_STEP3 + pr["train_steps"] * BYTES_PER_TRAIN_STEP3
    achieved = alg / (pr["walk_ms"] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "wave_geom_kernel + wave_dir_kernel (3D wavefront)",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_kind,
                "algorithmic_bytes_per_step": alg, "walk_ms_per_step": pr["walk_ms"],
                "train_ms_per_step": pr["train_ms"], "walk_steps_per_step": pr["steps"]}
    ncu_json = os.path.join(ROOT, "profiles", "ncu_counters_wave_geom_kernel.json")
    if os.path.exists(ncu_json):
        with open(ncu_json) as f:
            nc = json.load(f)
        roofline["traffic"] = nc.get("dram_bytes")
        roofline["traffic_source"] = os.path.relpath(ncu_json, ROOT)
    # e2e through the public API with host buffers
    field.set_state(p0, m0, v0, s0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.set_points(pts, offset)
    solver.run(SEED, wpp, train_until, tcfg)
    _ = solver.stats()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    quality = {"relmse_guided": rel_guided}
    if world == 1:  # uniform at equal samples
        us = Solver3(acc, None, abi.solver_config("uniform"))
        us.set_points(pts, offset)
        _, ums = us.run(SEED, wpp, 0, None)
        rel_u = relmse(us.stats()["mean"], ref)
        quality.update({"relmse_uniform_equal_wpp": rel_u, "vr_factor": rel_u / rel_guided if rel_guided else None,
                        "uniform_ms": ums, "uniform_walks_per_s": n_local * wpp / (ums * 1e-3)})
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        g, r = 48, 2
        c = cpu_oracle3_rate(g, r, r, os.cpu_count() or 1)
        cpu = {"value": c["value"], "unit": "walks/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{r} training wpp rounds of a {g}x{g} slice ({c['walks']} walks, {c['seconds']:.1f} s) "
                         f"through the 3D oracle port (no reference 3D code)"}
    if rank == 0:
        print(json.dumps({
            "metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(times)),
            "higher_is_better": True, "scaling": "strong" if cfg5 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: box-strip-vlin 3D (99,372 triangles), "
                                   f"{grid}x{grid if cfg5 else grid * world} slice, {wpp} wpp, learnable_mis, "
                                   f"training rounds < {train_until}",
                       "grid": [grid, grid if cfg5 else grid * world], "wpp": wpp, "train_until": train_until,
                       "mlp": "tensor (wavefront)", "l2": "flushed (256 MiB write) before every step",
                       "parallelism": f"dp{world} (points sharded, NCCL grad allreduce)"},
            "e2e": {"value": walks_per_step / e2e_s, "unit": "walks/s", "h2d_bytes_per_step": pts.nbytes,
                    "d2h_bytes_per_step": n_local * abi.POINT_STATS_DTYPE.itemsize},
            "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
            "walk_steps_per_s": pr["steps"] * world / (float(np.mean(times)) * 1e-3),
            "quality": quality}))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mlp", default="tensor", choices=["exact", "tensor"])
    ap.add_argument("--ref-rounds", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg4", "cfg5"])
    ap.add_argument("--grid", type=int, default=0, help="3D workloads: slice resolution (default 512 / 2048)")
    ap.add_argument("--wpp", type=int, default=0, help="3D workloads: walks per point (default 1024)")
    ap.add_argument("--train-until", type=int, default=TRAIN_UNTIL)
    args = ap.parse_args()
    if args.workload != "cfg2":
        return main3(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_2410_18944_b200 import _lib, abi, api
    from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse, analytic_image

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.init(local)

    preset = make_preset(PRESET)
    bb = preset.scene.bbox
    # weak scaling: rank r owns rows [GRID r, GRID (r+1)) of a GRID x GRID*world grid
    from paper_2410_18944_b200.parallel import broadcast_comm_id, shard_points
    all_pts = cell_centers(GRID, GRID * world, bb)
    n_local = GRID * GRID
    pts, offset = shard_points(all_pts, world, rank)

    fcfg = abi.field_config()
    field = api.GuidingField(fcfg, bb, SEED)
    p0, m0, v0, s0 = field.state()
    scfg = abi.solver_config("learnable_mis")
    solver = api.Solver(api.Accel(preset.scene), field, scfg,
                        api.MLP_TENSOR if args.mlp == "tensor" else api.MLP_EXACT)
    if world > 1:
        solver.attach_comm(broadcast_comm_id(dist, rank), world, rank)
    tcfg = abi.train_config(seed=SEED)
    solver.set_points(pts, offset)
    zero_stats = np.zeros(n_local, dtype=abi.POINT_STATS_DTYPE)
    l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one_step():
        field.set_state(p0, m0, v0, s0)  # every step trains from the same initial field
        solver.set_stats(zero_stats)
        flush_l2(l2)
        torch.cuda.synchronize()
        _, ms = solver.run(SEED, WPP, TRAIN_UNTIL, tcfg)
        return ms

    for _ in range(args.warmup):
        one_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    times, prof = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            times.append(one_step())
            prof.append(solver.run_profile())
    launches = (_lib.kernel_launches() - launches0) // max(1, args.steps)
    torch.cuda.synchronize()
    step_ms = float(np.mean(times))
    total_ms = float(np.sum(times))
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    walks_per_step = n_local * WPP * world
    value = walks_per_step * args.steps / (total_ms * 1e-3)

    # quality: relMSE of the last step against the analytic solution
    st = solver.stats()
    ref_img = np.array([preset.analytic(x, y) for x, y in pts])
    rel_guided = relmse(st["mean"], ref_img)

    # roofline of the dominant kernel (the walk kernel)
    pr = prof[-1]
    peaks, peak_kind = measured_peaks()
    alg_bytes = pr["steps"] * BYTES_PER_STEP + pr["train_steps"] * BYTES_PER_TRAIN_STEP
    achieved = alg_bytes / (pr["walk_ms"] * 1e-3) / 1e9
    kname = "walk_kernel_tc" if args.mlp == "tensor" else "walk_kernel_g8"
    # the walk phase of a round: the lockstep tile kernel plus, on small
    # scenes, the warp-per-walk kernel that finishes each CTA's last <= 24
    # walks (walk_kernel_coop_resume); walk_ms spans both
    klabel = kname + (" + walk_kernel_coop_resume (walk phase)" if args.mlp == "tensor" else "")
    rounds = max(1, WPP)
    roofline = {"bound": "hbm", "kernel": klabel, "achieved": achieved,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": None, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": alg_bytes / rounds,
                "algorithmic_bytes_per_step": alg_bytes, "walk_ms_per_step": pr["walk_ms"],
                "train_ms_per_step": pr["train_ms"], "walk_steps_per_step": pr["steps"]}
    # DRAM / L2 bytes of one launch of the same kernel from the committed ncu
    # --set full capture (profiles/, tools/ncu_counters.py): the walk state
    # lives in registers and the records stay in L2, so DRAM traffic is far
    # below the SoA algorithmic bytes; the kernel is latency-bound
    # (walk phase = lockstep kernel + tail resume kernel: bytes summed)
    names = [kname] + (["walk_kernel_coop_resume"] if args.mlp == "tensor" else [])
    files = [os.path.join(ROOT, "profiles", f"ncu_counters_{k}.json") for k in names]
    files = [f for f in files if os.path.exists(f)]
    if files:
        ncs = []
        for fn in files:
            with open(fn) as f:
                ncs.append(json.load(f))
        roofline["traffic"] = sum(nc.get("dram_bytes") or 0 for nc in ncs)
        roofline["traffic_source"] = " + ".join(os.path.relpath(fn, ROOT) for fn in files)
        roofline["l2_bytes_per_launch"] = sum(nc.get("l2_bytes") or 0 for nc in ncs)
        roofline["l2_gbs_achieved"] = ncs[0].get("l2_gbs")
        roofline["tensor_pipe_active_pct"] = ncs[0].get("tensor_pipe_active_pct")

    # e2e through the public API with host buffers (points in, statistics out)
    e2e_times = []
    h2d = pts.nbytes
    d2h = n_local * abi.POINT_STATS_DTYPE.itemsize
    for _ in range(max(1, min(2, args.steps))):
        field.set_state(p0, m0, v0, s0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.set_points(pts, offset)
        solver.run(SEED, WPP, TRAIN_UNTIL, tcfg)
        _ = solver.stats()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_times))
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # uniform WoSt at equal samples for the variance-reduction factor
    usolver = api.Solver(api.Accel(preset.scene), None, abi.solver_config("uniform"))
    usolver.set_points(pts, offset)
    usolver.run(SEED, WPP, 0, None)  # warm (allocations)
    usolver.set_stats(zero_stats)
    _, ums = usolver.run(SEED, WPP, 0, None)
    rel_uniform = relmse(usolver.stats()["mean"], ref_img)

    # estimator quality over 8 seeds (a single seed's relMSE scatters by ~10%):
    # guided (this arm's MLP path) and uniform at equal samples, and uniform at
    # equal device time (as many wpp as fit in the guided run's time)
    quality_seeds = []
    if world == 1:
        acc = api.Accel(preset.scene)
        # each solver is warmed by a short run (its first run allocates the
        # estimate buffers and record arena inside the timed window) and reset
        for sd in range(1, 9):
            f = api.GuidingField(abi.field_config(), preset.scene.bbox, sd)
            fs = f.state()
            gs = api.Solver(acc, f, abi.solver_config("learnable_mis"),
                            api.MLP_TENSOR if args.mlp == "tensor" else api.MLP_EXACT)
            gs.set_points(pts, offset)
            gs.run(sd, 2, 2, abi.train_config(seed=sd))
            f.set_state(*fs)
            gs.set_stats(zero_stats)
            _, gms = gs.run(sd, WPP, TRAIN_UNTIL, abi.train_config(seed=sd))
            us = api.Solver(acc, None, abi.solver_config("uniform"))
            us.set_points(pts, offset)
            us.run(sd, WPP, 0, None)
            us.set_stats(zero_stats)
            _, ums_s = us.run(sd, WPP, 0, None)
            quality_seeds.append((relmse(gs.stats()["mean"], ref_img), relmse(us.stats()["mean"], ref_img),
                                  gms, ums_s))
        q = np.array(quality_seeds)
        wpp_eq = int(WPP * q[:, 2].mean() / q[:, 3].mean())
        us = api.Solver(api.Accel(preset.scene), None, abi.solver_config("uniform"))
        us.set_points(pts, offset)
        us.run(SEED, wpp_eq, 0, None)
        us.set_stats(zero_stats)
        _, ums_eq = us.run(SEED, wpp_eq, 0, None)
        rel_uniform_eq_time = relmse(us.stats()["mean"], ref_img)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_rate(args.ref_rounds, os.cpu_count() or 1)
        if r:
            cpu = {"value": r["value"], "unit": "walks/s", "cores": os.cpu_count(),
                   "kind": r["kind"],
                   "sample": f"{args.ref_rounds} of {WPP} wpp rounds of the same workload "
                             f"({r['walks']} walks, {r['seconds']:.2f} s) via the reference's run_solve"}
    if rank == 0:
        line = {"metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"cfg2: {PRESET} {GRID}x{GRID * world} grid, {WPP} wpp, "
                                       f"learnable_mis, online training every round",
                           "preset": PRESET, "grid": [GRID, GRID * world], "wpp": WPP,
                           "train_until": TRAIN_UNTIL, "mlp": args.mlp,
                           "l2": "flushed (256 MiB write) before every step",
                           "parallelism": f"dp{world} (points sharded, NCCL grad allreduce)"},
                "e2e": {"value": walks_per_step / e2e_s, "unit": "walks/s",
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": int(launches),
                # walk steps per second: the walk kernel's steps of one
                # step (solve) over its device time, all ranks (weak scaling)
                "walk_steps_per_s": pr["steps"] * world / (step_ms * 1e-3),
                "roofline": roofline,
                "cpu_baseline": cpu,
                "clocks": clk.summary(),
                "quality": {"relmse_guided": rel_guided, "relmse_uniform_equal_wpp": rel_uniform,
                            "vr_factor": rel_uniform / rel_guided if rel_guided > 0 else None,
                            "uniform_ms": ums, "escaped": pr["escaped"]}}
        if quality_seeds:
            # reference side: tests/golden/ref_cfg2_seeds.json (its run_solve, seeds 1-8)
            q = np.array(quality_seeds)
            with open(os.path.join(ROOT, "tests", "golden", "ref_cfg2_seeds.json")) as f:
                rs = json.load(f)
            ref_g = float(np.mean(list(rs["learnable_mis"].values())))
            ref_u = float(np.mean(list(rs["uniform"].values())))
            line["quality"].update({
                "seeds": 8, "relmse_guided_mean": float(q[:, 0].mean()),
                "relmse_uniform_mean": float(q[:, 1].mean()),
                "vr_factor_mean": float(q[:, 1].mean() / q[:, 0].mean()),
                "reference_relmse_guided_mean_8seeds": ref_g, "reference_vr_factor_8seeds": ref_u / ref_g,
                "guided_ms_mean": float(q[:, 2].mean()), "uniform_ms_mean": float(q[:, 3].mean()),
                "uniform_equal_time_wpp": wpp_eq, "relmse_uniform_equal_time": rel_uniform_eq_time,
                "vr_factor_equal_time": rel_uniform_eq_time / float(q[:, 0].mean())})
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
