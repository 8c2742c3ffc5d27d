"""cfg 3 (BASELINE.json configs[2]): const-source-disk (256-gon unit disk,
f = 4, g = |x|^2 - 1, eps = 1e-6, analytic u = |x|^2 - 1), learnable MIS with
online training, against the analytic solution. Exercises the BVH walk path
(> 16 segments) and the Green's-ball source term.

  python tools/cfg3_check.py [--grid 128] [--wpp 256] [--seeds 1 2]

Prints one JSON line per (seed, mode, mlp) with relMSE, device ms, walks/s
and escapes.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=128)
    ap.add_argument("--wpp", type=int, default=256)
    ap.add_argument("--seeds", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--modes", nargs="+", default=["uniform", "tensor", "exact"])
    a = ap.parse_args()
    p = make_preset("const-source-disk")
    pts = cell_centers(a.grid, a.grid, p.eval_bbox)
    ref = np.array([p.analytic(x, y) for x, y in pts])
    acc = api.Accel(p.scene)
    for seed in a.seeds:
        for m in a.modes:
            if m == "uniform":
                s = api.Solver(acc, None, abi.solver_config("uniform"))
                s.set_points(pts)
                _, ms = s.run(seed, a.wpp, 0, None)
            else:
                f = api.GuidingField(abi.field_config(), p.scene.bbox, seed)
                s = api.Solver(acc, f, abi.solver_config("learnable_mis"),
                               api.MLP_TENSOR if m == "tensor" else api.MLP_EXACT)
                s.set_points(pts)
                _, ms = s.run(seed, a.wpp, 256, abi.train_config(seed=seed))
            st = s.stats()
            prof = s.run_profile()
            walks = len(pts) * a.wpp
            print(json.dumps({"seed": seed, "mode": m, "grid": a.grid, "wpp": a.wpp,
                              "relmse": relmse(st["mean"], ref), "ms": ms, "walks_per_s": walks / (ms * 1e-3),
                              "steps_per_walk": prof["steps"] / max(prof["walks"], 1),
                              "walk_ms": prof["walk_ms"], "train_ms": prof["train_ms"],
                              "escaped": int(st["escaped"].sum())}), flush=True)


if __name__ == "__main__":
    main()
