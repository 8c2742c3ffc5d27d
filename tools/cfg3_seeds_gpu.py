"""cfg 3 at 128^2 (const-source-disk, 256 wpp, learnable MIS trained every
round) over seeds on the GPU, through the 2D wavefront pair or the lockstep
kernel (WOSTGPU_WALK2): per-seed relMSE of guided and uniform as JSON lines.

  python tools/cfg3_seeds_gpu.py --seeds 32 --walk wave
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=32)
ap.add_argument("--walk", default="wave", choices=["wave", "lockstep"])
a = ap.parse_args()
os.environ["WOSTGPU_WALK2"] = a.walk
pr = make_preset("const-source-disk")
pts = cell_centers(128, 128, pr.eval_bbox)
truth = np.array([pr.analytic(x, y) for x, y in pts])
acc = api.Accel(pr.scene)
for seed in range(1, a.seeds + 1):
    t0 = time.time()
    f = api.GuidingField(abi.field_config(), pr.scene.bbox, seed)
    s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(pts)
    _, ms = s.run(seed, 256, 256, abi.train_config(seed=seed))
    print(json.dumps({"walk": a.walk, "seed": seed, "relmse": relmse(s.stats()["mean"], truth), "ms": ms,
                      "wall": time.time() - t0}), flush=True)
