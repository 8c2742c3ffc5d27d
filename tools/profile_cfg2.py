"""Short cfg-2 slice for profiling: a few guided training rounds plus a
uniform multi-round launch on the bench workload (neumann-strip-vlin 128^2)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--mlp", default="exact")
ap.add_argument("--uniform-rounds", type=int, default=16)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
p = make_preset("neumann-strip-vlin")
pts = cell_centers(128, 128, p.eval_bbox)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(api.Accel(p.scene), f, abi.solver_config("learnable_mis"),
               api.MLP_TENSOR if a.mlp == "tensor" else api.MLP_EXACT)
s.set_points(pts)
if a.warmup:
    s.run(1, 4, 256, abi.train_config(seed=1))  # module load, allocations
st, ms = s.run(1, a.rounds, 256, abi.train_config(seed=1))
prof = s.run_profile()
print(f"per round: walk {prof['walk_ms'] / a.rounds:.3f} ms, train {prof['train_ms'] / a.rounds:.3f} ms, "
      f"total {ms / a.rounds:.3f} ms")
est, esc, steps = s.walks()
print("guided", a.rounds, "rounds", round(ms, 3), "ms", prof)
print("last round steps: max", steps.max(), "mean", steps.mean(), "p99", np.percentile(steps, 99),
      "p999", np.percentile(steps, 99.9))
u = api.Solver(api.Accel(p.scene), None, abi.solver_config("uniform"))
u.set_points(pts)
_, ums = u.run(1, a.uniform_rounds, 0, None)
print("uniform", a.uniform_rounds, "rounds", round(ums, 3), "ms", u.run_profile())
