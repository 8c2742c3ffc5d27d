"""Diagnostic: exact-path guided walks and records vs the oracle on the
const-source-disk preset (source term), same field and seeds."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import Oracle  # noqa: E402
from paper_2410_18944_b200 import _lib, abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

_lib.init(0)
orc = Oracle("orc")
p = make_preset("const-source-disk")
cfg = abi.field_config()
fo = orc.field(cfg, p.scene.bbox, 31)
fg = api.GuidingField(cfg, p.scene.bbox, 31)
xy = cell_centers(24, 24, p.eval_bbox)
sc = abi.solver_config("learnable_mis")
ho = orc.scene(p.scene)
est_o, esc_o, _ = orc.walks(ho, fo, sc, xy, 7, 0)
sol = api.Solver(api.Accel(p.scene), fg, sc, api.MLP_EXACT)
sol.set_points(xy)
sol.solve_rounds(7, 0, 1)
est_g, esc_g, steps = sol.walks()
close = np.abs(est_o - est_g) <= 1e-9 * np.maximum(1.0, np.abs(est_o))
print("per-walk close fraction", close.mean(), "max diff", np.max(np.abs(est_o - est_g)))
st_o = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
rec_o = orc.solve_batch(ho, fo, sc, xy, st_o, 7, 0, collect=True)
sol2 = api.Solver(api.Accel(p.scene), fg, sc, api.MLP_EXACT)
st_g = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
rec_g = api.solve_batch(sol2, xy, st_g, 7, 0, collect_records=True)
print("records", len(rec_g), len(rec_o))
for k in ("target", "pdf_mis", "pdf_u"):
    a, b = np.sort(rec_g[k]), np.sort(rec_o[k])
    n = min(len(a), len(b))
    print(k, "max rel diff (sorted)", float(np.max(np.abs(a[:n] - b[:n]) / np.maximum(np.abs(b[:n]), 1e-6))),
          "sum ours/ref", float(a.sum()), float(b.sum()))
print("targets ours[:10]", np.sort(rec_g["target"])[-10:])
print("targets ref[:10] ", np.sort(rec_o["target"])[-10:])
