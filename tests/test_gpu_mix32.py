"""GPU parity of the tensor-core walk path's fp32 mixture math (wg_mix32.cuh)
against the oracle's fp64 restatement of sphdist.cpp: the Table-1 decode +
mixture pdf (normalize_params + mixture_pdf, sphdist.cpp:176-185, 287-310)
and the distribution of the fp32 Best-Fisher sampler (sphdist.cpp:120-140).

Tolerances: the decoded pdf agrees to 5e-5 relative wherever the oracle pdf
exceeds 1e-30 (fp32 exponent of |nu - mu|^2 form, log I0 polynomials to
2.5e-6); c to 1e-6. The sampler's angle histogram matches the oracle density
bin by bin (|z| < 5.5 for every bin expecting >= 50 samples, chi^2 tail
probability > 1e-5).
"""
import math

import numpy as np
import pytest
from scipy import stats

from paper_2410_18944_b200 import abi, api

pytestmark = pytest.mark.gpu


def _oracle_pdf(orc, raw32, nu2):
    m = orc.normalize(raw32.astype(np.float64), 8)
    f = orc.fn("mixture_pdf")
    out = np.empty(len(nu2))
    for i in range(len(nu2)):
        nu = np.array([nu2[i, 0], nu2[i, 1], 0.0])
        out[i] = f(abi.vptr(m[i:i + 1]), abi.ptr(nu))
    return out, m["c"]


def _raw_rows(rng, n):
    raw = rng.normal(0.0, 1.5, (n, 33))
    raw[:, 16:24] = rng.uniform(-16.0, 12.0, (n, 8))  # kappa from clamp-low to clamp-high
    raw[:8, 0:2] = 0.0  # zero-norm mean -> fallback direction
    return raw.astype(np.float32)


def test_mixture32_pdf_matches_oracle(gpu, orc):
    rng = np.random.default_rng(11)
    n = 3000
    raw = _raw_rows(rng, n)
    # directions: uniform, plus near the mode of a random lobe at ~1/sqrt(kappa)
    a = rng.uniform(-math.pi, math.pi, n)
    lobe = rng.integers(0, 8, n)
    mx, my = raw[np.arange(n), 2 * lobe], raw[np.arange(n), 2 * lobe + 1]
    kap = np.exp(np.clip(raw[np.arange(n), 16 + lobe].astype(np.float64), math.log(1e-6), math.log(1e4)))
    near = np.arctan2(my, mx) + rng.normal(0.0, 1.0, n) / np.sqrt(np.maximum(kap, 1.0))
    a = np.where(np.arange(n) % 2 == 0, a, near)
    nu = np.stack([np.cos(a), np.sin(a)], axis=1)
    pd, cd = api.mixture32_pdf(raw, nu)
    po, co = _oracle_pdf(orc, raw, nu)
    m = po > 1e-30
    rel = np.abs(pd[m] - po[m]) / po[m]
    assert rel.max() < 5e-5, (rel.max(), np.argmax(rel))
    np.testing.assert_allclose(cd, co, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("lobes", [
    [(0.3, 5.0, 0.6), (2.5, 2000.0, 0.4)],       # broad + very concentrated
    [(-1.0, 0.01, 0.5), (1.0, 40.0, 0.5)],       # almost uniform + medium
    [(0.0, 1e4, 1.0)],                           # clamp-high single lobe
])
def test_mixture32_sampler_distribution(gpu, orc, lobes):
    raw = np.zeros(33, dtype=np.float64)
    raw[24:32] = -30.0  # unused lobes get ~0 weight
    for i, (ang, kap, lam) in enumerate(lobes):
        raw[2 * i], raw[2 * i + 1] = math.cos(ang), math.sin(ang)
        raw[16 + i] = math.log(kap)
        raw[24 + i] = math.log(lam)
    raw32 = raw.astype(np.float32)
    n = 2_000_000
    nu = api.mixture32_sample(raw32, n, 2024)
    assert np.allclose(np.hypot(nu[:, 0], nu[:, 1]), 1.0, atol=1e-15)
    ang = np.arctan2(nu[:, 1], nu[:, 0])
    nb = 4096
    edges = np.linspace(-math.pi, math.pi, nb + 1)
    counts, _ = np.histogram(ang, edges)
    # expected bin probabilities from the oracle density (16-point midpoint rule)
    sub = 16
    mids = (edges[:-1, None] + (np.arange(sub)[None, :] + 0.5) * (edges[1] - edges[0]) / sub).ravel()
    m = orc.normalize(raw32.astype(np.float64)[None, :], 8)
    f = orc.fn("mixture_pdf")
    dens = np.array([f(abi.vptr(m), abi.ptr(np.array([math.cos(t), math.sin(t), 0.0]))) for t in mids])
    p = dens.reshape(nb, sub).mean(axis=1) * (edges[1] - edges[0])
    assert abs(p.sum() - 1.0) < 1e-3
    exp = p / p.sum() * n
    ok = exp >= 50
    z = (counts[ok] - exp[ok]) / np.sqrt(exp[ok])
    assert np.abs(z).max() < 5.5, np.abs(z).max()
    # chi^2 tail probability > 1e-5 (a fixed chi^2/dof bound is too tight for
    # the ~50 well-populated bins of the kappa = 1e4 lobe: sd of chi^2/dof 0.2)
    chi2 = float(np.sum(z ** 2))
    assert chi2 < stats.chi2.ppf(1.0 - 1e-5, int(ok.sum())), (chi2, int(ok.sum()))
    # mass outside the well-populated bins matches too
    assert abs(counts[~ok].sum() - exp[~ok].sum()) < 6.0 * math.sqrt(max(exp[~ok].sum(), 1.0)) + 5


def test_mixture3f_pdf_matches_oracle(gpu, orc):
    """The 3D direction kernel's fp32 decode + mixture density
    (wg3_mix32.cuh normalize3f / mixture_pdf3f) against the oracle's fp64
    d = 3 normalize_params + mixture_pdf: 5e-5 relative wherever the oracle
    pdf exceeds 1e-30, kappa from the clamp-low to the clamp-high end."""
    from paper_2410_18944_b200.api3 import mixture3f_pdf
    rng = np.random.default_rng(12)
    n = 4000
    raw = rng.normal(0.0, 1.5, (n, 41))
    raw[:, 24:32] = rng.uniform(-16.0, 12.0, (n, 8))  # log kappa
    raw[:8, 0:3] = 0.0  # zero-norm mean -> fallback direction
    raw = raw.astype(np.float32)
    # directions: uniform, plus near a random lobe's mean at ~1/sqrt(kappa)
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    lobe = rng.integers(0, 8, n)
    mu = raw[np.arange(n)[:, None], 3 * lobe[:, None] + np.arange(3)].astype(np.float64)
    mn = np.linalg.norm(mu, axis=1, keepdims=True)
    mu = np.where(mn > 1e-12, mu / np.maximum(mn, 1e-300), u)
    kap = np.exp(np.clip(raw[np.arange(n), 24 + lobe].astype(np.float64), math.log(1e-6), math.log(1e4)))
    near = mu + rng.normal(size=(n, 3)) / np.sqrt(np.maximum(kap, 1.0))[:, None]
    near /= np.linalg.norm(near, axis=1, keepdims=True)
    nu = np.where((np.arange(n) % 2 == 0)[:, None], u, near)
    pd, cd = mixture3f_pdf(raw, nu)
    m = orc.normalize(raw.astype(np.float64), 8, dim=3)
    f = orc.fn("mixture_pdf")
    po = np.array([f(abi.vptr(m[i:i + 1]), abi.ptr(np.ascontiguousarray(nu[i]))) for i in range(n)])
    ok = po > 1e-30
    rel = np.abs(pd[ok] - po[ok]) / po[ok]
    assert ok.sum() > n // 2 and rel.max() < 5e-5, (rel.max(), np.argmax(rel))
    np.testing.assert_allclose(cd, m["c"], rtol=1e-6, atol=1e-7)
