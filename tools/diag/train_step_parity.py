"""Diagnostic: one training call on identical records, reference (ref_ shim)
vs our device pipeline (train_batch), with the cap and minibatch large enough
that no random selection happens (one Adam step), then several steps."""
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
ref = Oracle("ref")
name = sys.argv[1] if len(sys.argv) > 1 else "const-source-disk"
p = make_preset(name)
cfg = abi.field_config()
fr = ref.field(cfg, p.scene.bbox, 31)
fg = api.GuidingField(cfg, p.scene.bbox, 31)
assert np.array_equal(ref.field_params(fr), fg.params())
xy = cell_centers(32, 32, p.eval_bbox)
sc = abi.solver_config("learnable_mis")
ho = ref.scene(p.scene)
st = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
recs = ref.solve_batch(ho, fr, sc, xy, st, 7, 0, collect=True)
print("records", len(recs))
for mlp in (api.MLP_EXACT, api.MLP_TENSOR):
    fg2 = api.GuidingField(cfg, p.scene.bbox, 31)
    fr2 = ref.field(cfg, p.scene.bbox, 31)
    sol = api.Solver(api.Accel(p.scene), fg2, sc, mlp)
    big = abi.train_config(minibatch=1 << 16, max_records=1 << 16, seed=1)
    for step in range(3):
        st_r = ref.train_batch(fr2, recs, big, step)
        st_g = sol.train_batch(recs, big, step)
        pr, pg = ref.field_params(fr2), fg2.params()
        d = np.abs(pr - pg)
        emb = 87040
        rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b - ref.field_params(ref.field(cfg, p.scene.bbox, 31))[: len(b)] if False else b), 1e-30)
        dp_r = pr - ref.field_params(ref.field(cfg, p.scene.bbox, 31))
        dp_g = pg - api.GuidingField(cfg, p.scene.bbox, 31).params()
        print(f"mlp {mlp} step {step}: consumed ref {st_r.records_consumed} ours {st_g.records_consumed}; "
              f"steps {st_r.steps}/{st_g.steps}; |dparams| ref {np.linalg.norm(dp_r):.4e} ours {np.linalg.norm(dp_g):.4e}; "
              f"|diff| {np.linalg.norm(pr - pg):.3e} max {d.max():.3e}; grad norm ref {st_r.mean_grad_norm:.4e} ours {st_g.mean_grad_norm:.4e}")
