"""Diagnostic: cfg 3 at 128^2, 256 rounds. (a) the fused wostgpu_run: which
points end non-finite; (b) host-driven rounds: first round with non-finite
estimates / params."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

p = make_preset("const-source-disk")
pts = cell_centers(128, 128, p.eval_bbox)
acc = api.Accel(p.scene)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
s.set_points(pts)
s.run(1, 256, 256, abi.train_config(seed=1))
st = s.stats()
bad = np.where(~np.isfinite(st["mean"]))[0]
print("run: non-finite points", len(bad), bad[:10], "params finite", bool(np.all(np.isfinite(f.params()))))
if len(bad):
    print("  xy", pts[bad[:5]], "count", st["count"][bad[:5]], "m2", st["m2"][bad[:5]])
f2 = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s2 = api.Solver(acc, f2, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
s2.set_points(pts)
tc = abi.train_config(seed=1)
for r in range(256):
    s2.solve_rounds(1, r, 1, collect=True)
    est, esc, steps = s2.walks()
    if not np.all(np.isfinite(est)):
        i = np.where(~np.isfinite(est))[0]
        recs = s2.records()
        print("round", r, "non-finite estimates", len(i), "points", i[:5], pts[i[:5]], "steps", steps[i[:5]])
        w = recs[np.isin(np.arange(len(recs)), np.arange(len(recs)))]
        print("  records non-finite:", {k: int(np.sum(~np.isfinite(recs[k]))) for k in ["target", "pdf_mis", "pdf_g", "pdf_u", "c"]},
              "min pdf_mis", float(np.nanmin(recs["pdf_mis"])))
        break
    s2.train_round(tc, r)
    if not np.all(np.isfinite(f2.params())):
        print("round", r, "params non-finite after training")
        break
else:
    print("host-driven: all 256 rounds finite")
