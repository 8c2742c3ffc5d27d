"""Diagnostic: find the cfg-3 training records whose (tensor-core) gradient is
non-finite, by bisection with field_grad, and print their raw MLP outputs."""
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
tc = abi.train_config(seed=1)


def finite_grad(recs):
    g = s.field_grad(recs, tc)
    return bool(np.all(np.isfinite(g))), g


for r in range(256):
    s.solve_rounds(1, r, 1, collect=True)
    recs = s.records()
    use = recs[(recs["pdf_mis"] >= tc.pdf_floor) & (recs["target"] >= 0)]
    ok, g = finite_grad(use)
    if not ok:
        print("round", r, "records", len(use), "non-finite grad entries", int(np.sum(~np.isfinite(g))))
        bad = use
        while len(bad) > 1:
            h = len(bad) // 2
            a_ok, _ = finite_grad(bad[:h])
            bad = bad[h:] if a_ok else bad[:h]
        print("offending record:", bad)
        xy = np.array([bad["x"][0][:2]])
        for mlp in (api.MLP_EXACT, api.MLP_TENSOR):
            print("raw MLP outputs", mlp, np.array2string(f.eval_batch(xy, mlp)[0], precision=4))
        s2 = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_EXACT)
        s2.set_points(pts)
        ok2, _ = (lambda g2: (bool(np.all(np.isfinite(g2))), g2))(s2.field_grad(bad, tc))
        print("exact-path gradient finite:", ok2)
        break
    s.train_round(tc, r)
else:
    print("no non-finite gradient in 256 rounds")
