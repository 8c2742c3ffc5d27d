"""One device-timed solve per BASELINE.json configuration (for BASELINE.md
§5): walks/s, walk-steps/s, relMSE against the analytic solution, and the
uniform solve of the same points (VR). cfg 5 runs on one GPU.

  python tools/measure_cfgs.py [--skip-cfg5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.api3 import MLP_TENSOR, Accel3, GuidingField3, Solver3  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse  # noqa: E402
from paper_2410_18944_b200.scene3 import make_preset3, slice_points, strip_vlin_np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--skip-cfg5", action="store_true")
a = ap.parse_args()


def two_d(name, preset, grid, wpp):
    p = make_preset(preset)
    pts = cell_centers(grid, grid, p.eval_bbox)
    truth = np.array([p.analytic(x, y) for x, y in pts])
    acc = api.Accel(p.scene)
    out = {"config": name, "grid": grid, "wpp": wpp}
    for mode in ("uniform", "learnable_mis"):
        f = api.GuidingField(abi.field_config(), p.scene.bbox, 1) if mode != "uniform" else None
        s = api.Solver(acc, f, abi.solver_config(mode), api.MLP_TENSOR)
        s.set_points(pts)
        tc = abi.train_config(seed=1) if f else None
        s.run(1, 2 if f else wpp, 2 if f else 0, tc)  # warm-up: allocations (uniform: the full round buffer)
        if f:
            f2 = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
            s = api.Solver(acc, f2, abi.solver_config(mode), api.MLP_TENSOR)
            s.set_points(pts)
            s.run(1, 2, 2, tc)
            f2.set_state(*api.GuidingField(abi.field_config(), p.scene.bbox, 1).state())
        s.set_stats(np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE))
        _, ms = s.run(1, wpp, 256 if f else 0, tc)
        pr = s.run_profile()
        out[mode] = {"walks_per_s": len(pts) * wpp / (ms * 1e-3), "steps_per_s": pr["steps"] / (ms * 1e-3),
                     "ms": ms, "relmse": relmse(s.stats()["mean"], truth)}
    out["vr"] = out["uniform"]["relmse"] / out["learnable_mis"]["relmse"]
    print(json.dumps(out), flush=True)


def three_d(name, grid, wpp):
    p = make_preset3("box-strip-vlin")
    pts = slice_points(grid, grid)
    truth = strip_vlin_np(pts[:, 0], pts[:, 1])
    acc = Accel3(p.scene)
    out = {"config": name, "grid": grid, "wpp": wpp}
    for mode in ("uniform", "learnable_mis"):
        f = GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), 1) if mode != "uniform" else None
        s = Solver3(acc, f, abi.solver_config(mode), MLP_TENSOR)
        s.set_points(pts)
        tc = abi.train_config(seed=1) if f else None
        s.run(1, 2, 2 if f else 0, tc)  # warm-up: module load, slot pool, record arena
        if f:
            f.set_state(*GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), 1).state())
        _, ms = s.run(1, wpp, 256 if f else 0, tc)
        pr = s.run_profile()
        out[mode] = {"walks_per_s": len(pts) * wpp / (ms * 1e-3), "steps_per_s": pr["steps"] / (ms * 1e-3),
                     "ms": ms, "relmse": relmse(s.stats()["mean"], truth)}
    out["vr"] = out["uniform"]["relmse"] / out["learnable_mis"]["relmse"]
    print(json.dumps(out), flush=True)


two_d("cfg1+cfg2", "neumann-strip-vlin", 128, 256)
two_d("cfg3", "const-source-disk", 512, 256)
three_d("cfg4", 512, 1024)
if not a.skip_cfg5:
    three_d("cfg5 (one GPU)", 2048, 1024)
