"""Diagnostic: cfg-3 training round by round on the tensor-core path; report
the first round whose parameters, estimates or records are non-finite."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

mlp = api.MLP_TENSOR if (len(sys.argv) < 2 or sys.argv[1] == "tensor") else api.MLP_EXACT
p = make_preset("const-source-disk")
pts = cell_centers(64, 64, p.eval_bbox)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(api.Accel(p.scene), f, abi.solver_config("learnable_mis"), mlp)
s.set_points(pts)
tc = abi.train_config(seed=1)
for r in range(64):
    s.solve_rounds(1, r, 1, collect=True)
    est, esc, steps = s.walks()
    recs = s.records()
    bad_est = int(np.sum(~np.isfinite(est)))
    fields = ["target", "pdf_mis", "pdf_g", "pdf_u", "c"]
    bad_rec = {k: int(np.sum(~np.isfinite(recs[k]))) for k in fields}
    st = s.train_round(tc, r)
    prm = f.params()
    bad_p = int(np.sum(~np.isfinite(prm)))
    print(r, "est_nonfinite", bad_est, "rec_nonfinite", bad_rec, "max target", float(np.nanmax(recs["target"])) if len(recs) else 0,
          "min pdf_mis", float(np.nanmin(recs["pdf_mis"])) if len(recs) else 0, "grad_norm", st.mean_grad_norm,
          "params_nonfinite", bad_p, "max|p|", float(np.nanmax(np.abs(prm))), flush=True)
    if bad_p or bad_est:
        i = np.where(~np.isfinite(est))[0][:5]
        print("bad points", i, pts[i] if len(i) else "", "steps", steps[i] if len(i) else "")
        break
