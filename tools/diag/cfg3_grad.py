"""Diagnostic: minibatch gradient parity (oracle fp64 vs ours) on records of
the const-source-disk preset, for a fresh and for a GPU-trained field."""
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
p = make_preset(sys.argv[1] if len(sys.argv) > 1 else "const-source-disk")
cfg = abi.field_config()
fo = orc.field(cfg, p.scene.bbox, 31)
fg = api.GuidingField(cfg, p.scene.bbox, 31)
xy = cell_centers(40, 40, p.eval_bbox)
sc = abi.solver_config("learnable_mis")
ho = orc.scene(p.scene)
tc = abi.train_config(seed=1)
acc = api.Accel(p.scene)
for phase in ("fresh", "trained"):
    if phase == "trained":  # train on the GPU, copy the params to the oracle field
        s = api.Solver(acc, fg, sc, api.MLP_TENSOR)
        s.set_points(cell_centers(128, 128, p.eval_bbox))
        s.run(1, 32, 256, tc)
        orc.field_set_params(fo, fg.params())
    st = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
    recs = orc.solve_batch(ho, fo, sc, xy, st, 7, 0, collect=True)[:8192]
    g_o = orc.field_grad(fo, recs, tc)
    for mlp in (api.MLP_EXACT, api.MLP_TENSOR):
        sol = api.Solver(acc, fg, sc, mlp)
        g_g = sol.field_grad(recs, tc)
        emb = 87040
        errs = [np.linalg.norm(g_g[sl] - g_o[sl]) / max(np.linalg.norm(g_o[sl]), 1e-300)
                for sl in (slice(0, emb), slice(emb, None))]
        print(phase, "mlp", mlp, "rel L2 err emb %.3e mlp %.3e" % tuple(errs), "|g| %.3e" % np.linalg.norm(g_o))
