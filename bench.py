"""Benchmark: guided walk-on-stars walks/s on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[3], "cfg 4", the largest
single-GPU configuration of the metric's 1/2/4/8-GPU sweep): box-strip-vlin,
the unit box as 99,372 triangles (Dirichlet x = 0 / x = 1, insulated lateral
faces), a 512 x 512 slice at z = 0.5 per GPU, 1024 walks per point,
learnable-MIS guiding trained online in the first 256 rounds. One step = one
complete solve (1024 wpp rounds, the first 256 each followed by a training
round) = 268,435,456 walks per GPU.

Second block in the same JSON line, "cfg2" (BASELINE.json configs[1], the
configuration anchored to the reference's own C++ implementation): preset
neumann-strip-vlin (proj/src/presets.cpp:217-221), 128 x 128 grid per GPU,
256 wpp, learnable MIS trained every round; fully timed with the same
--steps / --warmup, its own roofline, e2e, cpu_baseline (the reference's
run_solve on the host cores, all 256 rounds) and relMSE at equal time vs
that CPU reference.

  python bench.py [--gpus N --steps K --warmup W]       our CUDA path
  python bench.py --impl reference [...]                the reference on host cores
  python bench.py --workload cfg2|cfg5 [...]            one workload alone

N > 1: one rank per GPU (torchrun; a plain `python bench.py --gpus N`
re-executes itself under torch.distributed.run). Weak scaling: rank r owns
rows [r H, (r+1) H) of an H x (H N) grid over the same domain (the global
point index keys every walk's stream); guiding-field training is global
(usable-record count and every minibatch's gradient sum allreduced with NCCL
over NVLink), so all ranks take identical Adam steps.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 1
TRAIN_UNTIL = 256
# cfg 2 (2D)
PRESET = "neumann-strip-vlin"
GRID = 128
WPP = 256
# algorithmic HBM bytes per walk step: 52 B SoA walk state read
# + written = 104 B; training rounds add a 56 B trace record written + read
BYTES_PER_STEP = 104
BYTES_PER_TRAIN_STEP = 112
FLOP_PER_EVAL2 = 14464   # 2 (16*64 + 64*64 + 64*33)
FLOP_PER_RECORD2 = 43392  # forward + dX + dW
# cfg 4 / 5 (3D): 60 B SoA state read + written = 120 B; +68 B record w + r
BYTES_PER_STEP3 = 120
BYTES_PER_TRAIN_STEP3 = 136
FLOP_PER_EVAL3 = 15488   # 2 (16*64 + 64*64 + 64*41)
DTYPE = "f64+f32+f16mma"
DTYPE_DETAIL = ("walk state, geometry and estimates in f64; guiding-mixture math in f32; guiding MLP "
                "on tcgen05 tensor cores with f16 operands (split hi/lo) and f32 accumulation; "
                "training gradients f32, Adam moments f64")


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1350.0}, "fallback"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


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


def ncu_counters(names):
    """Per-launch DRAM / L2 bytes of the named kernels from the committed
    ncu --set full captures (profiles/ncu_counters_<kernel>.json)."""
    files = [os.path.join(ROOT, "profiles", f"ncu_counters_{k}.json") for k in names]
    files = [f for f in files if os.path.exists(f)]
    if not files:
        return {}
    ncs = []
    for fn in files:
        with open(fn) as f:
            ncs.append(json.load(f))
    out = {"traffic": sum(nc.get("dram_bytes") or 0 for nc in ncs),
           "traffic_source": " + ".join(os.path.relpath(fn, ROOT) for fn in files),
           "l2_bytes_per_launch": sum(nc.get("l2_bytes") or 0 for nc in ncs),
           "l2_gbs_achieved": ncs[0].get("l2_gbs"),
           "tensor_pipe_active_pct": ncs[0].get("tensor_pipe_active_pct")}
    cfgs = {nc.get("config") for nc in ncs if nc.get("config")}
    if cfgs:
        out["traffic_config"] = " / ".join(sorted(cfgs))
    return out


def max_over_ranks(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU side
def cpu_reference_run(rounds, threads, mode=3, preset=PRESET, grid=GRID, train_until=TRAIN_UNTIL):
    """The reference's own run_solve (oracle/_ref, built from /root/reference
    with its Release flags) on the host cores: `rounds` wpp rounds of the
    workload. Returns seconds (RunResult.seconds) and relMSE vs analytic."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_FAST_SO, REF_SO, Oracle
    so = REF_FAST_SO if os.path.exists(REF_FAST_SO) else REF_SO
    if not os.path.exists(so):
        return None
    os.environ["OMP_NUM_THREADS"] = str(threads)
    os.environ["WOST_THREADS"] = str(threads)
    ref = Oracle("ref", so)
    sec, rel, tsec = (np.zeros(1) for _ in range(3))
    import ctypes as C
    rc = ref.lib.ref_run_solve(preset.encode(), grid, grid, rounds, mode, train_until, SEED, None,
                               sec.ctypes.data_as(C.POINTER(C.c_double)),
                               rel.ctypes.data_as(C.POINTER(C.c_double)),
                               tsec.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        return None
    walks = grid * grid * rounds
    return {"value": walks / float(sec[0]), "seconds": float(sec[0]), "relmse": float(rel[0]),
            "train_seconds": float(tsec[0]), "walks": walks, "kind": "reference",
            "so": os.path.relpath(so, ROOT)}


# cfg 4 CPU sample: the 3D oracle port (the reference has no 3D code) on a
# G x G slice for R rounds, the first R/4 of them training (the full
# workload's 256 : 768 split of training to frozen rounds)
# 3D oracle-port samples of the cfg 4 workload (same domain, slice and 1:3
# training : frozen split): the product arm's cpu_baseline is one sample of
# ~10 s of host work; the reference arm times a smaller sample per step so
# its whole --steps K --warmup W run stays within a few minutes
CPU3_GRID, CPU3_ROUNDS = 128, 104
REF3_GRID, REF3_ROUNDS = 96, 16


def cpu_oracle3_run(grid, rounds, train_until, threads):
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
    return {"value": walks / sec, "seconds": sec, "walks": walks, "kind": "port", "grid": grid, "rounds": rounds}


def cpu3_sample_text(c):
    g, r = c["grid"], c["rounds"]
    return (f"{r} wpp rounds ({r // 4} training, {r - r // 4} frozen: "
            f"the workload's 1:3 split) of a {g}x{g} slice of the cfg 4 domain "
            f"({c['walks']} walks, {c['seconds']:.1f} s) through the 3D oracle port "
            f"(oracle/wost3d.inc; the reference has no 3D code)")


def run_reference(args):
    """--impl reference: the reference's CPU implementation on the host cores.
    Headline = the workload's CPU sample; cfg 2 = the reference's own
    run_solve on the full configuration (all 256 rounds: same config)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    base = {"metric": "guided WoSt walks/sec", "unit": "walks/s", "impl": "reference", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "host_cpu": cpu_model()}

    rounds = args.ref_rounds

    def cfg2_block(steps, warmup):
        for _ in range(warmup):
            cpu_reference_run(rounds, threads)
        rr = [cpu_reference_run(rounds, threads) for _ in range(steps)]
        if any(r is None for r in rr):
            return None
        v = float(np.mean([r["value"] for r in rr]))
        return {"value": v, "unit": "walks/s", "ms_per_step": float(np.mean([r["seconds"] for r in rr])) * 1e3,
                "steps": steps, "warmup": warmup, "same_config": rounds == WPP,
                "relmse": float(np.mean([r["relmse"] for r in rr])),
                "train_seconds": float(np.mean([r["train_seconds"] for r in rr])),
                "config": {"workload": f"cfg2: {PRESET} {GRID}x{GRID} grid, {WPP} wpp, learnable_mis, "
                                       f"online training every round (reference run_solve, {rounds} of "
                                       f"{WPP} rounds)"},
                "cpu_baseline": {"value": v, "unit": "walks/s", "cores": threads, "kind": "reference",
                                 "sample": f"cfg 2 solve, {rounds} of {WPP} rounds, via the reference's run_solve "
                                           f"({rr[0]['so']})"}}

    if args.workload == "cfg2":
        b = cfg2_block(args.steps, args.warmup)
        if b is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        line = dict(base, **b, scaling="weak")
        line["e2e"] = {"value": b["value"], "unit": "walks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
        print(json.dumps(line))
        return
    # cfg 4 / 5: the 3D oracle port on a bounded sample
    for _ in range(args.warmup):
        cpu_oracle3_run(REF3_GRID, REF3_ROUNDS, REF3_ROUNDS // 4, threads)
    rr = [cpu_oracle3_run(REF3_GRID, REF3_ROUNDS, REF3_ROUNDS // 4, threads) for _ in range(args.steps)]
    value = float(np.mean([x["value"] for x in rr]))
    line = dict(base, value=value, ms_per_step=float(np.mean([x["seconds"] for x in rr])) * 1e3,
                scaling="strong" if args.workload == "cfg5" else "weak",
                config={"workload": f"{args.workload} oracle-port sample {REF3_GRID}x{REF3_GRID} x "
                                    f"{REF3_ROUNDS} wpp"},
                cpu_baseline={"value": value, "unit": "walks/s", "cores": threads, "kind": "port",
                              "sample": cpu3_sample_text(rr[0])},
                e2e={"value": value, "unit": "walks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    b = None if args.no_cfg2 else cfg2_block(min(args.steps, 3), min(args.warmup, 1))
    if b is not None:
        line["cfg2"] = b
    print(json.dumps(line))


# ---------------------------------------------------------------- cfg 2 (2D)
def bench_cfg2(args, dist, world, rank, local):
    """cfg 2 on this rank's 128 x 128 shard: timed solves, e2e, roofline,
    estimator quality, and (rank 0, N = 1) the reference on the host cores."""
    import torch
    from paper_2410_18944_b200 import _lib, abi, api
    from paper_2410_18944_b200.parallel import broadcast_comm_id, shard_points
    from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse

    preset = make_preset(PRESET)
    bb = preset.scene.bbox
    all_pts = cell_centers(GRID, GRID * world, bb)
    n_local = GRID * GRID
    pts, offset = shard_points(all_pts, world, rank)
    mlp = api.MLP_TENSOR if args.mlp == "tensor" else api.MLP_EXACT
    field = api.GuidingField(abi.field_config(), bb, SEED)
    p0, m0, v0, s0 = field.state()
    acc = api.Accel(preset.scene)
    solver = api.Solver(acc, field, abi.solver_config("learnable_mis"), mlp)
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
    step_ms = float(np.mean(times))
    total_ms = max_over_ranks(dist, float(np.sum(times)))
    walks_per_step = n_local * WPP * world
    value = walks_per_step * args.steps / (total_ms * 1e-3)
    truth = np.array([preset.analytic(x, y) for x, y in pts])
    rel_guided = relmse(solver.stats()["mean"], truth)

    pr = prof[-1]
    peaks, peak_kind = measured_peaks()
    alg_bytes = pr["steps"] * BYTES_PER_STEP + pr["train_steps"] * BYTES_PER_TRAIN_STEP
    achieved = alg_bytes / (pr["walk_ms"] * 1e-3) / 1e9
    kname = "walk_kernel_tc" if args.mlp == "tensor" else "walk_kernel_g8"
    # the walk phase of a round: the lockstep tile kernel plus, on small
    # scenes, the warp-per-walk kernel that finishes each CTA's last <= 24
    # walks (walk_kernel_coop_resume); walk_ms spans both
    names = [kname] + (["walk_kernel_coop_resume"] if args.mlp == "tensor" else [])
    mlp_tflops = pr["steps"] * FLOP_PER_EVAL2 / (pr["walk_ms"] * 1e-3) / 1e12
    train_tflops = pr["train_steps"] * FLOP_PER_RECORD2 / max(pr["train_ms"] * 1e-3, 1e-9) / 1e12
    roofline = {"bound": "hbm", "kernel": " + ".join(names) + " (walk phase, one launch pair per round)",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": alg_bytes / WPP,
                "algorithmic_bytes_per_step": alg_bytes, "walk_ms_per_step": pr["walk_ms"],
                "train_ms_per_step": pr["train_ms"], "walk_steps_per_step": pr["steps"],
                "tensor": {"mlp_tflops_over_walk_phase": mlp_tflops,
                           "train_tflops_over_train_phase": train_tflops,
                           "peak_tflops_sustained": peaks.get("bf16_tflops_sustained"),
                           "frac_walk": mlp_tflops / peaks.get("bf16_tflops_sustained", 1365.0)}}
    roofline.update(ncu_counters(names))

    # critical path of a lockstep round: a round ends with its longest walk
    # (one walk per point, rounds do not overlap), so the walk phase is
    # bounded below by (longest walk's steps) x (latency of one dependent
    # step), not by HBM. Longest walks sampled over 16 rounds of the trained
    # field.
    longest = []
    for r in range(16):
        solver.solve_rounds(SEED + 100, r, 1)
        longest.append(int(solver.walks()[2].max()))
    walk_ms_round = pr["walk_ms"] / WPP
    crit = {"longest_walk_steps_mean": float(np.mean(longest)), "longest_walk_steps_max": int(max(longest)),
            "mean_steps_per_walk": pr["steps"] / (n_local * WPP),
            "walk_ms_per_round": walk_ms_round,
            "us_per_critical_step": walk_ms_round * 1e3 / float(np.mean(longest)),
            "note": "a lockstep round lasts as long as its longest walk: walk_ms_per_round / "
                    "longest_walk_steps = achieved latency per dependent walk step"}

    # e2e through the public API with host buffers (points in, statistics out)
    e2e_times = []
    h2d = pts.nbytes
    d2h = n_local * abi.POINT_STATS_DTYPE.itemsize
    for _ in range(max(1, min(3, args.steps))):
        field.set_state(p0, m0, v0, s0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver.set_points(pts, offset)
        solver.run(SEED, WPP, TRAIN_UNTIL, tcfg)
        _ = solver.stats()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(dist, float(np.mean(e2e_times)))

    usolver = api.Solver(acc, None, abi.solver_config("uniform"))
    usolver.set_points(pts, offset)
    usolver.run(SEED, WPP, 0, None)  # warm (allocations)
    usolver.set_stats(zero_stats)
    _, ums = usolver.run(SEED, WPP, 0, None)
    rel_uniform = relmse(usolver.stats()["mean"], truth)
    quality = {"relmse_guided": rel_guided, "relmse_uniform_equal_wpp": rel_uniform,
               "vr_factor": rel_uniform / rel_guided if rel_guided > 0 else None,
               "uniform_ms": ums, "escaped": pr["escaped"]}

    block = {"metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s", "n_gpus": world,
             "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
             "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
             "config": {"workload": f"cfg2: {PRESET} {GRID}x{GRID * world} grid, {WPP} wpp, "
                                    f"learnable_mis, online training every round",
                        "preset": PRESET, "grid": [GRID, GRID * world], "wpp": WPP,
                        "train_until": TRAIN_UNTIL, "mlp": args.mlp,
                        "l2": "flushed (256 MiB write) before every step",
                        "parallelism": f"dp{world} (points sharded, global training, NCCL allreduce)"},
             "e2e": {"value": walks_per_step / e2e_s, "unit": "walks/s", "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": d2h},
             "gpu_launches": int(launches),
             "walk_steps_per_s": pr["steps"] * world / (step_ms * 1e-3),
             "roofline": roofline, "critical_path": crit, "clocks": clk.summary(), "quality": quality}

    if world == 1:
        # estimator quality over 8 seeds (one seed's relMSE scatters ~10%):
        # guided and uniform at equal samples, uniform at equal device time
        qs = []
        for sd in range(1, 9):
            f = api.GuidingField(abi.field_config(), bb, sd)
            fs = f.state()
            gs = api.Solver(acc, f, abi.solver_config("learnable_mis"), mlp)
            gs.set_points(pts, offset)
            gs.run(sd, 2, 2, abi.train_config(seed=sd))  # warm: allocations
            f.set_state(*fs)
            gs.set_stats(zero_stats)
            _, gms = gs.run(sd, WPP, TRAIN_UNTIL, abi.train_config(seed=sd))
            us = api.Solver(acc, None, abi.solver_config("uniform"))
            us.set_points(pts, offset)
            us.run(sd, WPP, 0, None)
            us.set_stats(zero_stats)
            _, ums_s = us.run(sd, WPP, 0, None)
            qs.append((relmse(gs.stats()["mean"], truth), relmse(us.stats()["mean"], truth), gms, ums_s))
        q = np.array(qs)
        wpp_eq = int(WPP * q[:, 2].mean() / q[:, 3].mean())
        us = api.Solver(acc, None, abi.solver_config("uniform"))
        us.set_points(pts, offset)
        us.run(SEED, wpp_eq, 0, None)
        us.set_stats(zero_stats)
        us.run(SEED, wpp_eq, 0, None)
        rel_u_eq = relmse(us.stats()["mean"], truth)
        with open(os.path.join(ROOT, "tests", "golden", "ref_cfg2_seeds.json")) as fh:
            rs = json.load(fh)
        ref_g = float(np.mean(list(rs["learnable_mis"].values())))
        ref_u = float(np.mean(list(rs["uniform"].values())))
        quality.update({
            "seeds": 8, "relmse_guided_mean": float(q[:, 0].mean()),
            "relmse_uniform_mean": float(q[:, 1].mean()),
            "vr_factor_mean": float(q[:, 1].mean() / q[:, 0].mean()),
            "reference_relmse_guided_mean_8seeds": ref_g, "reference_vr_factor_8seeds": ref_u / ref_g,
            "guided_ms_mean": float(q[:, 2].mean()), "uniform_ms_mean": float(q[:, 3].mean()),
            "uniform_equal_time_wpp": wpp_eq, "relmse_uniform_equal_time": rel_u_eq,
            "vr_factor_equal_time_gpu_uniform": rel_u_eq / float(q[:, 0].mean())})

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rg = cpu_reference_run(WPP, threads, mode=3)
        ru = cpu_reference_run(WPP, threads, mode=0)
        if rg:
            block["cpu_baseline"] = {
                "value": rg["value"], "unit": "walks/s", "cores": threads, "kind": "reference",
                "sample": f"the full cfg 2 solve ({WPP} rounds, {rg['walks']} walks, {rg['seconds']:.2f} s) "
                          f"via the reference's run_solve ({rg['so']})", "host_cpu": cpu_model()}
            # relMSE at equal time vs the CPU reference: the
            # GPU guided solve gets the CPU reference's wall time for this
            # configuration; wpp beyond 256 are frozen-field rounds
            f = api.GuidingField(abi.field_config(), bb, SEED)
            fs = f.state()
            gs = api.Solver(acc, f, abi.solver_config("learnable_mis"), mlp)
            gs.set_points(pts, offset)
            gs.run(SEED, 2, 2, abi.train_config(seed=SEED))
            f.set_state(*fs)
            gs.set_stats(zero_stats)
            _, t512 = gs.run(SEED, 2 * WPP, TRAIN_UNTIL, tcfg)
            per_round = max((t512 - step_ms) / WPP, 1e-3)

            def equal_time(target_s):
                w = int(min(1 << 16, WPP + max(0.0, target_s * 1e3 - step_ms) / per_round))
                f.set_state(*fs)
                gs.set_stats(zero_stats)
                _, ms = gs.run(SEED, w, TRAIN_UNTIL, tcfg)
                return w, ms, relmse(gs.stats()["mean"], truth)

            w, ms, rel = equal_time(rg["seconds"])
            et = {"cpu_reference_guided_s": rg["seconds"], "cpu_reference_guided_relmse": rg["relmse"],
                  "gpu_guided_wpp_in_that_time": w, "gpu_guided_ms": ms, "gpu_guided_relmse": rel,
                  "relmse_ratio_cpu_over_gpu": rg["relmse"] / rel if rel > 0 else None}
            if ru:
                w2, ms2, rel2 = equal_time(ru["seconds"])
                et.update({"cpu_reference_uniform_s": ru["seconds"], "cpu_reference_uniform_relmse": ru["relmse"],
                           "gpu_guided_wpp_in_uniform_time": w2, "gpu_guided_ms_uniform_time": ms2,
                           "gpu_guided_relmse_uniform_time": rel2,
                           "relmse_ratio_cpu_uniform_over_gpu": ru["relmse"] / rel2 if rel2 > 0 else None})
            quality["equal_time_vs_cpu_reference"] = et
    return block


# ---------------------------------------------------------------- cfg 4 / 5 (3D)
def bench_cfg3d(args, dist, world, rank, local):
    import torch
    from paper_2410_18944_b200 import _lib, abi
    from paper_2410_18944_b200.api3 import Accel3, GuidingField3, MLP_TENSOR, Solver3
    from paper_2410_18944_b200.parallel import broadcast_comm_id, shard_points
    from paper_2410_18944_b200.scene import relmse
    from paper_2410_18944_b200.scene3 import make_preset3, slice_points, strip_vlin_np

    cfg5 = args.workload == "cfg5"
    grid = args.grid or (2048 if cfg5 else 512)
    wpp = args.wpp or 1024
    train_until = min(args.train_until, wpp)
    preset = make_preset3("box-strip-vlin")
    # cfg 5: strong scaling, the fixed 2048^2 slice split over ranks; cfg 4:
    # weak scaling, rank r owns rows [grid r, grid (r+1)) of a grid x grid*world slice
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
    total_ms = max_over_ranks(dist, float(np.sum(times)))
    step_ms = float(np.mean(times))
    walks_per_step = len(all_pts) * wpp
    value = walks_per_step * args.steps / (total_ms * 1e-3)
    truth = strip_vlin_np(pts[:, 0], pts[:, 1])
    rel_guided = relmse(solver.stats()["mean"], truth)
    pr = prof[-1]
    peaks, peak_kind = measured_peaks()
    alg = pr["steps"] * BYTES_PER_STEP3 + pr["train_steps"] * BYTES_PER_TRAIN_STEP3
    achieved = alg / (pr["walk_ms"] * 1e-3) / 1e9
    mlp_tflops = pr["steps"] * FLOP_PER_EVAL3 / (pr["walk_ms"] * 1e-3) / 1e12
    roofline = {"bound": "hbm", "kernel": "wave_geom_kernel + wave_dir_kernel (3D wavefront walk phase)",
                "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_kind,
                "algorithmic_bytes_per_step": alg, "walk_ms_per_step": pr["walk_ms"],
                "train_ms_per_step": pr["train_ms"], "walk_steps_per_step": pr["steps"],
                "bytes_per_walk_step": BYTES_PER_STEP3,
                "tensor": {"mlp_tflops_over_walk_phase": mlp_tflops,
                           "peak_tflops_sustained": peaks.get("bf16_tflops_sustained"),
                           "frac_walk": mlp_tflops / peaks.get("bf16_tflops_sustained", 1365.0)}}
    roofline.update(ncu_counters(["wave_geom_kernel"]))
    if roofline.get("l2_bytes_per_launch") and roofline.get("traffic_config"):
        roofline["note"] = ("traffic / l2 bytes are per wave_geom_kernel launch of the ncu capture named in "
                            "traffic_config; a launch advances every live slot by one geometry stage")
    # e2e through the public API with host buffers
    field.set_state(p0, m0, v0, s0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solver.set_points(pts, offset)
    solver.run(SEED, wpp, train_until, tcfg)
    _ = solver.stats()
    e2e_s = max_over_ranks(dist, time.perf_counter() - t0)
    quality = {"relmse_guided": rel_guided}
    if world == 1:  # uniform at equal samples and at equal device time
        us = Solver3(acc, None, abi.solver_config("uniform"))
        us.set_points(pts, offset)
        _, ums = us.run(SEED, wpp, 0, None)
        rel_u = relmse(us.stats()["mean"], truth)
        wpp_eq = int(wpp * step_ms / ums)
        _, ums_eq = us.run(SEED, wpp_eq, 0, None)
        rel_u_eq = relmse(us.stats()["mean"], truth)
        quality.update({"relmse_uniform_equal_wpp": rel_u, "vr_factor": rel_u / rel_guided if rel_guided else None,
                        "uniform_ms": ums, "uniform_walks_per_s": n_local * wpp / (ums * 1e-3),
                        "uniform_equal_time_wpp": wpp_eq, "uniform_equal_time_ms": ums_eq,
                        "relmse_uniform_equal_time": rel_u_eq,
                        "vr_factor_equal_time": rel_u_eq / rel_guided if rel_guided else None})
    block = {
        "metric": "guided WoSt walks/sec", "value": value, "unit": "walks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "strong" if cfg5 else "weak", "vs_baseline": None,
        "dtype": DTYPE, "dtype_detail": DTYPE_DETAIL, "data": "synthetic",
        "config": {"workload": f"{args.workload}: box-strip-vlin 3D (99,372 triangles), "
                               f"{grid}x{grid if cfg5 else grid * world} slice, {wpp} wpp, learnable_mis, "
                               f"training rounds < {train_until}",
                   "grid": [grid, grid if cfg5 else grid * world], "wpp": wpp, "train_until": train_until,
                   "mlp": "tensor (wavefront)", "l2": "flushed (256 MiB write) before every step",
                   "parallelism": f"dp{world} (points sharded, global training, NCCL allreduce)"},
        "e2e": {"value": walks_per_step / e2e_s, "unit": "walks/s", "h2d_bytes_per_step": pts.nbytes,
                "d2h_bytes_per_step": n_local * abi.POINT_STATS_DTYPE.itemsize},
        "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": None, "clocks": clk.summary(),
        "walk_steps_per_s": pr["steps"] * world / (step_ms * 1e-3),
        "mean_steps_per_walk": pr["steps"] / (n_local * wpp), "quality": quality}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_oracle3_run(CPU3_GRID, CPU3_ROUNDS, CPU3_ROUNDS // 4, os.cpu_count() or 1)
        block["cpu_baseline"] = {"value": c["value"], "unit": "walks/s", "cores": os.cpu_count(), "kind": "port",
                                 "sample": cpu3_sample_text(c), "host_cpu": cpu_model()}
    return block


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without a torchrun environment: re-execute
    this script with one rank per GPU (the driver's own launch line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mlp", default="tensor", choices=["exact", "tensor"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg4", choices=["cfg2", "cfg4", "cfg5"])
    ap.add_argument("--no-cfg2", action="store_true", help="cfg4/cfg5: skip the cfg 2 block")
    ap.add_argument("--grid", type=int, default=0, help="3D workloads: slice resolution (default 512 / 2048)")
    ap.add_argument("--wpp", type=int, default=0, help="3D workloads: walks per point (default 1024)")
    ap.add_argument("--train-until", type=int, default=TRAIN_UNTIL)
    ap.add_argument("--ref-rounds", type=int, default=WPP,
                    help="--impl reference, cfg 2: wpp rounds per step (default: all 256, the full config)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"

    import torch
    from paper_2410_18944_b200 import _lib
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.init(local)
    if args.workload == "cfg2":
        line = bench_cfg2(args, dist, world, rank, local)
        line.update({"data": "synthetic", "dtype_detail": DTYPE_DETAIL})
    else:
        line = bench_cfg3d(args, dist, world, rank, local)
        if not args.no_cfg2:
            line["cfg2"] = bench_cfg2(args, dist, world, rank, local)
    line["nccl_nranks"] = world if world > 1 else 0
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
