"""Diagnostic: binned z-scores of the fp32 sampler vs scipy's exact von Mises
and vs the oracle density used by tests/test_gpu_mix32.py (kappa = 1e4)."""
import math
import os
import sys

import numpy as np
from scipy import stats

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2410_18944_b200 import _lib, abi, api  # noqa: E402
from oracle_lib import Oracle  # noqa: E402

_lib.init(0)
orc = Oracle("orc")
kap = float(sys.argv[1]) if len(sys.argv) > 1 else 1e4
raw = np.zeros(33)
raw[24:32] = -30.0
raw[0], raw[1] = 1.0, 0.0
raw[16] = math.log(kap)
raw[24] = 0.0
raw32 = raw.astype(np.float32)
n = 2_000_000
nb = 4096
edges = np.linspace(-math.pi, math.pi, nb + 1)
sub = 16
mids = (edges[:-1, None] + (np.arange(sub)[None, :] + 0.5) * (edges[1] - edges[0]) / sub).ravel()
m = orc.normalize(raw32.astype(np.float64)[None, :], 8)
f = orc.fn("mixture_pdf")
dens = np.array([f(abi.vptr(m), abi.ptr(np.array([math.cos(t), math.sin(t), 0.0]))) for t in mids])
p = dens.reshape(nb, sub).mean(axis=1) * (edges[1] - edges[0])
exp = p / p.sum() * n
ok = exp >= 50


def report(name, ang):
    c, _ = np.histogram(ang, edges)
    z = (c[ok] - exp[ok]) / np.sqrt(exp[ok])
    print(f"{name}: chi2/dof {np.sum(z**2) / ok.sum():.3f} dof {ok.sum()} max|z| {np.abs(z).max():.2f}")
    idx = np.where(ok)[0]
    print("  z by bin:", " ".join(f"{edges[i]:+.4f}:{zz:+.1f}" for i, zz in zip(idx, z)))


nu = api.mixture32_sample(raw32, n, 2024)
report("gpu fp32", np.arctan2(nu[:, 1], nu[:, 0]))
k64 = float(m["kappa"][0, 0])
report("scipy vonmises", stats.vonmises.rvs(k64, size=n, random_state=np.random.default_rng(5)))
print("kappa oracle", k64)
# duplicates / stream correlation
u, cnt = np.unique(nu, axis=0, return_counts=True)
print("distinct samples", len(u), "of", n, "max multiplicity", cnt.max())
