"""Estimator-quality comparison on cfg 2 (neumann-strip-vlin 128^2, 256 wpp):
relMSE against the analytic solution for several seeds, uniform vs guided
(exact-arithmetic and tensor-core paths), plus per-point agreement with the
reference's own statistics (tests/golden/ref_cfg2_*.npz) in standard errors.

  python tools/quality_cfg2.py [--seeds 1 2 3 4] [--wpp 256]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse  # noqa: E402


def se(st):
    c = st["count"].astype(np.float64)
    return np.sqrt(np.where(c > 1, st["m2"] / (c * (c - 1)), 0.0))


def zfrac(a_mean, a_se, b_mean, b_se, k=3.0):
    s = np.sqrt(a_se ** 2 + b_se ** 2)
    return float(np.mean(np.abs(a_mean - b_mean) > k * np.maximum(s, 1e-300)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, nargs="+", default=[1, 2, 3, 4])
    ap.add_argument("--wpp", type=int, default=256)
    ap.add_argument("--grid", type=int, default=128)
    a = ap.parse_args()
    pr = make_preset("neumann-strip-vlin")
    pts = cell_centers(a.grid, a.grid, pr.eval_bbox)
    ref_img = np.array([pr.analytic(x, y) for x, y in pts])
    acc = api.Accel(pr.scene)
    out = {"grid": a.grid, "wpp": a.wpp, "runs": []}
    golden = {}
    for mode in ("uniform", "learnable"):
        path = os.path.join(ROOT, "tests", "golden", f"ref_cfg2_{mode}_seed1.npz")
        if os.path.exists(path):
            golden[mode] = np.load(path)
    for seed in a.seeds:
        for mode, mlp in (("uniform", None), ("learnable_mis", api.MLP_EXACT),
                          ("learnable_mis", api.MLP_TENSOR)):
            field = None
            if mode != "uniform":
                field = api.GuidingField(abi.field_config(), pr.scene.bbox, seed)
            s = api.Solver(acc, field, abi.solver_config(mode), mlp if mlp is not None else 1)
            s.set_points(pts)
            st, ms = s.run(seed, a.wpp, 256, abi.train_config(seed=seed) if field else None)
            stats = s.stats()
            row = {"seed": seed, "mode": mode, "mlp": {None: "-", 0: "exact", 1: "tensor"}[mlp],
                   "relmse": relmse(stats["mean"], ref_img), "ms": ms,
                   "escaped": int(stats["escaped"].sum())}
            key = "uniform" if mode == "uniform" else "learnable"
            if seed == 1 and key in golden and a.grid == 128 and a.wpp == 256:
                g = golden[key]
                row["frac_beyond_3se_vs_reference"] = zfrac(stats["mean"], se(stats), g["mean"],
                                                             g["se"])
                if key == "uniform":
                    row["max_abs_diff_vs_reference"] = float(np.max(np.abs(stats["mean"] - g["mean"])))
            out["runs"].append(row)
            print(json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
