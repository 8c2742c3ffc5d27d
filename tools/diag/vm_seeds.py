"""Diagnostic: chi^2/dof of the fp32 sampler (kappa = 1e4) over several seeds."""
import math
import os
import sys

import numpy as np
from scipy.special import i0e

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_18944_b200 import _lib, api  # noqa: E402

_lib.init(0)
for kap in (1e4, 40.0):
    raw = np.zeros(33)
    raw[24:32] = -30.0
    raw[0], raw[1] = 1.0, 0.0
    raw[16] = math.log(kap)
    raw[24] = 0.0
    n = 2_000_000
    edges = np.linspace(-math.pi, math.pi, 4097)
    sub = 64
    w = edges[1] - edges[0]
    mids = edges[:-1, None] + (np.arange(sub)[None, :] + 0.5) * w / sub
    p = (np.exp(kap * (np.cos(mids) - 1)) / (2 * math.pi * i0e(kap))).mean(axis=1) * w
    e = p / p.sum() * n
    ok = e >= 50
    vals = []
    for seed in range(1, 13):
        nu = api.mixture32_sample(raw.astype(np.float32), n, seed)
        c, _ = np.histogram(np.arctan2(nu[:, 1], nu[:, 0]), edges)
        z = (c[ok] - e[ok]) / np.sqrt(e[ok])
        vals.append((z ** 2).mean())
    print(f"kappa {kap}: dof {ok.sum()} chi2/dof per seed", " ".join(f"{v:.2f}" for v in vals),
          f"mean {np.mean(vals):.3f}")
