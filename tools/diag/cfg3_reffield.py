"""Diagnostic: the reference-trained cfg-3 field (WGF1 from its run_solve):
decoded c / kappa statistics, and our guided walks with that fixed field."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

p = make_preset("const-source-disk")
pts = cell_centers(128, 128, p.eval_bbox)
ref = np.array([p.analytic(x, y) for x, y in pts])
acc = api.Accel(p.scene)
fr = api.GuidingField.load(os.path.join(ROOT, "diag_data", "ref_cfg3_field_s1.wgf"))
mix = api.normalize_params(fr.eval_batch(pts, api.MLP_EXACT), 8)
print(f"reference field: adam steps {fr.state()[3]}; c mean {mix['c'].mean():.3f} max {mix['c'].max():.4f} "
      f"min {mix['c'].min():.3f}; kappa max {mix['kappa'].max():.1f}")
maxabs = np.max(np.abs(ref))
for mlp in (api.MLP_EXACT, api.MLP_TENSOR):
    for seed in (1, 2):
        s = api.Solver(acc, fr, abi.solver_config("learnable_mis"), mlp)
        s.set_points(pts)
        s.run(seed, 256, 0, None)  # fixed field: no training
        st = s.stats()
        e = (st["mean"] - ref) ** 2 / (ref ** 2 + 1e-4 * maxabs ** 2)
        print(f"our walks, reference field fixed, mlp {mlp} seed {seed}: relmse {e.mean():.5f}")
# and our own trained field, same protocol (train, then fixed-field walks)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
s.set_points(pts)
s.run(1, 256, 256, abi.train_config(seed=1))
mix = api.normalize_params(f.eval_batch(pts, api.MLP_EXACT), 8)
print(f"our field: c mean {mix['c'].mean():.3f} max {mix['c'].max():.4f} min {mix['c'].min():.3f}; "
      f"kappa max {mix['kappa'].max():.1f}")
for seed in (1, 2):
    s2 = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s2.set_points(pts)
    s2.run(seed + 10, 256, 0, None)
    st = s2.stats()
    e = (st["mean"] - ref) ** 2 / (ref ** 2 + 1e-4 * maxabs ** 2)
    print(f"our walks, our field fixed, seed {seed + 10}: relmse {e.mean():.5f}")
