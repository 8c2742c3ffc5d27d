"""3D throughput probe (cfg 4 shape): box-strip-vlin (n = 91, 99,372
triangles), a G x G slice at z = 0.5, uniform and guided (learnable MIS,
training every round until --train-until) runs; prints walks/s, steps/walk,
relMSE against the analytic solution.

  python tools/profile3.py [--grid 128] [--wpp 64] [--train-until 64]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_18944_b200 import abi  # noqa: E402
from paper_2410_18944_b200.api3 import Accel3, GuidingField3, Solver3  # noqa: E402
from paper_2410_18944_b200.scene3 import analytic_slice, make_preset3, slice_points  # noqa: E402
from paper_2410_18944_b200.scene import relmse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--wpp", type=int, default=64)
ap.add_argument("--train-until", type=int, default=64)
ap.add_argument("--modes", nargs="+", default=["uniform", "learnable_mis"])
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
p = make_preset3("box-strip-vlin")
x = slice_points(a.grid, a.grid)
ref = analytic_slice(p, a.grid, a.grid)
acc = Accel3(p.scene)
for m in a.modes:
    f = None if m == "uniform" else GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), a.seed)
    s = Solver3(acc, f, abi.solver_config(m))
    s.set_points(x)
    s.run(a.seed, 2, 0, None)  # warm-up (module load, allocations)
    if f is not None:
        f = GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), a.seed)
        s = Solver3(acc, f, abi.solver_config(m))
        s.set_points(x)
    st, ms = s.run(a.seed, a.wpp, a.train_until if f else 0, abi.train_config(seed=a.seed) if f else None)
    prof = s.run_profile()
    walks = len(x) * a.wpp
    print(json.dumps({"mode": m, "grid": a.grid, "wpp": a.wpp, "ms": ms, "walks_per_s": walks / (ms * 1e-3),
                      "steps_per_walk": prof["steps"] / max(prof["walks"], 1), "walk_ms": prof["walk_ms"],
                      "train_ms": prof["train_ms"], "relmse": relmse(s.stats()["mean"], ref),
                      "escaped": prof["escaped"], "train_steps": st.steps}), flush=True)
