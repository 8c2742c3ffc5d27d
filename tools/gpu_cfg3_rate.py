"""cfg 3 throughput at 512^2 (2D wavefront pair): guided learnable MIS over
R rounds, walks/s and walk ms. python tools/gpu_cfg3_rate.py [rounds]"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse  # noqa: E402
R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = make_preset("const-source-disk")
pts = cell_centers(512, 512, p.eval_bbox)
truth = np.array([p.analytic(x, y) for x, y in pts])
acc = api.Accel(p.scene)
for train_until in (R, 0):
    f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
    s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(pts)
    s.run(1, 2, 2, abi.train_config(seed=1))
    s.set_stats(np.zeros(len(pts), dtype=abi.POINT_STATS_DTYPE))
    _, ms = s.run(1, R, train_until, abi.train_config(seed=1))
    print(json.dumps({"train_until": train_until, "rounds": R, "ms": ms, "walks_per_s": len(pts) * R / (ms * 1e-3),
                      "relmse": relmse(s.stats()["mean"], truth)}))
