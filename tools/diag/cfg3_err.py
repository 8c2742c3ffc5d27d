"""Diagnostic: where the cfg-3 guided error sits (per-point contributions to
relMSE) and what the trained field decodes to (c, kappa) at the eval points."""
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
for seed in (1, 2):
    f = api.GuidingField(abi.field_config(), p.scene.bbox, seed)
    s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(pts)
    st_tr, ms = s.run(seed, 256, 256, abi.train_config(seed=seed))
    st = s.stats()
    maxabs = np.max(np.abs(ref))
    e = (st["mean"] - ref) ** 2 / (ref ** 2 + 1e-4 * maxabs ** 2)
    o = np.argsort(e)[::-1]
    print(f"seed {seed}: relmse {e.mean():.5f}, top-10 share {e[o[:10]].sum() / e.sum():.3f}, median {np.median(e):.2e}")
    se = np.sqrt(st["m2"] / (st["count"] * (st["count"] - 1)))
    for i in o[:5]:
        print(f"   pt {pts[i]} est {st['mean'][i]:.4f} ref {ref[i]:.4f} se {se[i]:.4f} contrib {e[i] / e.sum():.3f}")
    raw = f.eval_batch(pts, api.MLP_EXACT)
    mix = api.normalize_params(raw, 8)
    c = mix["c"]
    kap = mix["kappa"]
    print(f"   c: mean {c.mean():.3f} max {c.max():.3f} min {c.min():.3f}; kappa max {kap.max():.1f}, "
          f"frac lobes kappa>100 {np.mean(kap > 100):.3f}; train steps {st_tr.steps} consumed {st_tr.records_consumed} "
          f"skipped_v {st_tr.skipped_low_v}")
