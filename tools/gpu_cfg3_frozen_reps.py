"""cfg 3 frozen-round timing repeated in one process (outlier hunt):
python tools/gpu_cfg3_frozen_reps.py [reps] [rounds]"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
p = make_preset("const-source-disk")
pts = cell_centers(512, 512, p.eval_bbox)
acc = api.Accel(p.scene)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
s.set_points(pts)
s.run(1, 2, 2, abi.train_config(seed=1))
out = []
for i in range(reps):
    s.set_stats(np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE))
    _, ms = s.run(1 + i, R, 0, abi.train_config(seed=1))
    prof = s.run_profile()
    out.append(round(ms, 1))
    print(json.dumps({"rep": i, "ms": ms, "walk_ms": prof["walk_ms"], "steps": prof["steps"], "launches": prof.get("launches")}), flush=True)
print("TAIL2", os.environ.get("WOSTGPU_WAVE2_TAIL"), out)
