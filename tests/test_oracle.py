"""CPU suite: the oracle restatement (oracle/liboracle.so) pinned against
  * golden vectors generated from the reference library itself
    (tests/golden/*.npz, tests/golden/make_golden.py),
  * the reference library directly when oracle/_ref is built here,
  * the reference unit tests' known answers (proj/tests/*.cpp)."""
import hashlib
import math
import os

import numpy as np
import pytest

from fixtures import Rng, probes, random_scene
from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.scene import PRESET_NAMES, cell_centers, make_preset

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(G, name))


# ---------------------------------------------------------------- golden
def test_geometry_matches_reference_golden(orc):
    g = load("geometry.npz")
    h = orc.scene(random_scene(Rng(101, 0), 1000))
    for kinds in (1, 2, 3):
        pt, d, seg = orc.closest_point(h, g["cp_xy"], kinds)
        assert np.array_equal(seg, g[f"cp_seg_{kinds}"])
        assert np.array_equal(d, g[f"cp_d_{kinds}"])
        assert np.array_equal(pt, g[f"cp_pt_{kinds}"])
    assert np.array_equal(orc.closest_silhouette(h, g["cp_xy"]), g["sil_d"])
    t, p, n, s, k = orc.ray_first_hit(h, g["ray_o"], g["ray_d"], 2.0, 3)
    for a, b in ((t, "ray_t"), (p, "ray_p"), (n, "ray_n"), (s, "ray_seg"), (k, "ray_kind")):
        assert np.array_equal(a, g[b])
    assert orc.fn("t_epsilon")(h) == g["t_eps"][0]


def test_field_matches_reference_golden(orc):
    g = load("field.npz")
    f = orc.field(abi.field_config(), (0.0, 0.0, 1.0, 1.0), 1234)
    p = orc.field_params(f)
    assert hashlib.sha256(p.tobytes()).digest() == bytes(g["sha256"])
    assert np.array_equal(orc.field_eval(f, g["xy"], 33), g["out"])


def test_walks_match_reference_golden(orc):
    g = load("walks.npz")
    cfg = abi.field_config()
    for name in ("neumann-strip-vlin", "harmonic-disk", "curves"):
        pr = make_preset(name)
        h = orc.scene(pr.scene)
        xy = g[f"{name}_xy"]
        est, esc, nrec = orc.walks(h, None, abi.solver_config("uniform"), xy, 1, 0, records=True)
        assert np.array_equal(est, g[f"{name}_uniform"])
        assert np.array_equal(esc, g[f"{name}_uniform_esc"])
        assert np.array_equal(nrec, g[f"{name}_uniform_steps"])
        f = orc.field(cfg, pr.scene.bbox, 7)
        est, _, _ = orc.walks(h, f, abi.solver_config("learnable_mis"), xy, 1, 0)
        assert np.array_equal(est, g[f"{name}_guided"])


def test_training_matches_reference_golden(orc):
    g = load("train.npz")
    pr = make_preset("curves")
    h = orc.scene(pr.scene)
    f = orc.field(abi.field_config(), pr.scene.bbox, 31)
    st = np.zeros(400, dtype=abi.POINT_STATS_DTYPE)
    recs = orc.solve_batch(h, f, abi.solver_config("learnable_mis"), cell_centers(20, 20, pr.eval_bbox),
                           st, 7, 0, collect=True)
    assert np.array_equal(recs, g["recs"])
    assert np.array_equal(st["mean"], g["stats_mean"]) and np.array_equal(st["m2"], g["stats_m2"])
    tc = abi.train_config(seed=1)
    grad = orc.field_grad(f, recs[:1024], tc)
    np.testing.assert_allclose(grad, g["grad"], rtol=1e-12, atol=1e-18)
    ts = orc.train_batch(f, recs, tc, 0)
    assert ts.records_consumed == g["consumed"] and ts.steps == g["steps"]
    assert ts.mean_grad_norm == pytest.approx(float(g["norm"]), rel=1e-12)
    assert hashlib.sha256(orc.field_params(f).tobytes()).digest() == bytes(g["after_sha"])


# ---------------------------------------------------------------- vs reference
def test_oracle_bit_exact_with_reference_library(orc, ref):
    for seed, n in (((55, 1), 500), ((77, 3), 3000)):
        sc = random_scene(Rng(*seed), n)
        ho, hr = orc.scene(sc), ref.scene(sc)
        xy = probes(Rng(seed[0], 9), 2000, -0.2, 1.2)
        for kinds in (1, 2, 3):
            for a, b in zip(orc.closest_point(ho, xy, kinds), ref.closest_point(hr, xy, kinds)):
                assert np.array_equal(a, b)
        assert np.array_equal(orc.closest_silhouette(ho, xy), ref.closest_silhouette(hr, xy))
    for name in PRESET_NAMES:
        pr = make_preset(name)
        ho, hr = orc.scene(pr.scene), ref.scene(pr.scene)
        xy = cell_centers(24, 24, pr.eval_bbox)
        for mode in ("uniform", "fixed_mis"):
            fo = orc.field(abi.field_config(), pr.scene.bbox, 3) if mode != "uniform" else None
            fr = ref.field(abi.field_config(), pr.scene.bbox, 3) if mode != "uniform" else None
            a = orc.walks(ho, fo, abi.solver_config(mode), xy, 5, 2)
            b = ref.walks(hr, fr, abi.solver_config(mode), xy, 5, 2)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_oracle_flux_and_raster_scenes_bit_exact_with_reference(orc, ref):
    """Neumann flux (sample_neumann_contrib, wost.cpp:89-109) and raster
    values / source (scene.cpp:13-20, 53-67): the restatement reproduces the
    reference's walks bit for bit, uniform and guided."""
    from fixtures import flux_scene, raster_scene
    xy = cell_centers(20, 20, (0.1, 0.1, 0.9, 0.9))
    for sc in (flux_scene(), raster_scene()):
        ho, hr = orc.scene(sc), ref.scene(sc)
        assert orc.fn("has_neumann_flux")(ho) == ref.fn("has_neumann_flux")(hr)
        for mode in ("uniform", "learnable_mis"):
            fo = orc.field(abi.field_config(), sc.bbox, 4) if mode != "uniform" else None
            fr = ref.field(abi.field_config(), sc.bbox, 4) if mode != "uniform" else None
            a = orc.walks(ho, fo, abi.solver_config(mode), xy, 6, 1)
            b = ref.walks(hr, fr, abi.solver_config(mode), xy, 6, 1)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert np.std(a[0]) > 0
    # raster values evaluated on the host mirror RasterGrid::at
    g = raster_scene().values[0]
    assert g.eval(-0.3, 0.5) == g.raster[2, 0] and g.eval(0.999, 1.7) == g.raster[4, 6]


# ---------------------------------------------------------------- unit KATs
def test_bessel_known_answers(orc):
    # proj/tests/test_sphdist.cpp:62-76
    i0 = orc.fn("bessel_i0")
    assert i0(1.0) == pytest.approx(1.2660658777520084, rel=1e-10)
    assert i0(10.0) == pytest.approx(2815.7166284662544, rel=1e-10)
    assert i0(50.0) == pytest.approx(2.9325537838493457e20, rel=1e-9)
    assert math.exp(orc.fn("log_bessel_i0")(100.0)) == pytest.approx(1.0737517071310738e42, rel=1e-9)
    r = orc.fn("bessel_i1_over_i0")
    assert r(1.0) == pytest.approx(0.4463899658965345, rel=1e-10)
    assert r(12.0) == pytest.approx(0.9573814053952422, rel=1e-9)
    assert r(25.0) == pytest.approx(0.9797914534905159, rel=1e-9)


def test_normalisation_table1(orc):
    # proj/tests/test_sphdist.cpp:441-461
    raw = np.zeros((1, 4 * 2 + 1))
    raw[0, 0:2] = (3.0, 4.0)
    raw[0, 2:4] = (0.0, 0.0)  # zero-norm -> fallback direction of index 1
    raw[0, 4] = math.log(2.0)
    raw[0, 5] = 20.0  # exp(20) clamps to 1e4
    raw[0, 6:8] = (0.0, math.log(3.0))
    raw[0, 8] = 0.0
    m = orc.normalize(raw, 2)[0]
    assert np.allclose(m["mu"][0], (0.6, 0.8, 0.0))
    a = 2 * math.pi * 1 / 16
    assert np.allclose(m["mu"][1], (math.cos(a), math.sin(a), 0.0))
    assert m["kappa"][0] == pytest.approx(2.0) and m["kappa"][1] == 1e4
    assert m["lambda"][0] == pytest.approx(0.25) and m["lambda"][1] == pytest.approx(0.75)
    assert m["c"] == 0.5


def test_vmf_peak_and_mis_pdf(orc):
    # vmf_pdf(mu | mu, kappa = 1) = 0.341710 (test_sphdist.cpp:86-94)
    m = np.zeros(1, dtype=abi.MIXTURE_DTYPE)
    m["k"], m["dim"], m["c"] = 1, 2, 0.5
    m["mu"][0, 0] = (1.0, 0.0, 0.0)
    m["kappa"][0, 0], m["lambda"][0, 0] = 1.0, 1.0
    nu = np.array([1.0, 0.0, 0.0])
    p = orc.fn("mixture_pdf")(abi.vptr(m), abi.ptr(nu))
    assert p == pytest.approx(0.341710, rel=1e-5)
    # mis_pdf = c p_g + (1 - c) p_u
    pm = orc.fn("mis_pdf")(abi.vptr(m), abi.ptr(nu), None, 1)
    assert pm == pytest.approx(0.5 * p + 0.5 / (2 * math.pi), rel=1e-12)
    # zero on or below the tangent plane of a Neumann boundary
    n = np.array([0.0, 1.0, 0.0])
    below = np.array([0.0, -1.0, 0.0])
    assert orc.fn("mis_pdf")(abi.vptr(m), abi.ptr(below), abi.ptr(n), 1) == 0.0


def test_constant_boundary_is_reproduced_exactly(orc):
    # proj/tests/test_wost.cpp:339-349 (maximum principle, bit-exact 0.75)
    from fixtures import polygon_scene
    sc = polygon_scene((0.0, 0.0), 1.0, 32, abi.DIRICHLET, 0.75, (-1.1, -1.1, 1.1, 1.1))
    h = orc.scene(sc)
    xy = np.tile([[0.1, -0.2]], (2000, 1))
    est, esc, _ = orc.walks(h, None, abi.solver_config("uniform"), xy, 13, 0,
                            point_index=np.arange(2000))
    assert np.all(est == 0.75) and not esc.any()


def test_harmonic_disk_unbiased(orc):
    # proj/tests/test_wost.cpp:312-322: mean at (0.3, 0.2) is 0.05 within 3 SE
    pr = make_preset("harmonic-disk")
    h = orc.scene(pr.scene)
    n = 20000
    est, _, _ = orc.walks(h, None, abi.solver_config("uniform"), np.tile([[0.3, 0.2]], (n, 1)), 11, 0,
                          point_index=np.arange(n))
    se = est.std(ddof=1) / math.sqrt(n)
    assert abs(est.mean() - 0.05) < 3 * se


def test_d3_mixture_and_gradient_match_reference(orc, ref):
    """The d = 3 vMF pieces the 3D path builds on, oracle vs the reference
    library: Table-1 normalisation (sphdist.cpp:287-310), mixture and MIS
    densities with and without a Neumann normal (:176-270), and the
    raw-parameter gradient through a mixture_dim = 3 field (mixture_grad with
    dlogv_dkappa's d = 3 branch, sphdist.cpp:315-381; kl_grad /
    selection_grad, guide_train.cpp:25-56). Plus the reference test's d = 3
    vMF peak (kappa = 2: 0.324236, proj/tests/test_sphdist.cpp)."""
    rng = np.random.default_rng(17)
    raw = rng.normal(scale=1.5, size=(40, 41))
    mo, mr = orc.normalize(raw, 8, 3), ref.normalize(raw, 8, 3)
    for k in ("mu", "kappa", "lambda", "log_a", "c"):
        np.testing.assert_allclose(mo[k], mr[k], rtol=1e-14, atol=1e-300)
    for i in range(len(raw)):
        nu = rng.normal(size=3)
        nu /= np.linalg.norm(nu)
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        a = orc.fn("mixture_pdf")(abi.vptr(mo[i:i + 1]), abi.ptr(nu))
        b = ref.fn("mixture_pdf")(abi.vptr(mr[i:i + 1]), abi.ptr(nu))
        assert a == pytest.approx(b, rel=1e-13)
        for normal in (None, n):
            a = orc.fn("mis_pdf")(abi.vptr(mo[i:i + 1]), abi.ptr(nu), None if normal is None else abi.ptr(normal), 1)
            b = ref.fn("mis_pdf")(abi.vptr(mr[i:i + 1]), abi.ptr(nu), None if normal is None else abi.ptr(normal), 1)
            assert a == pytest.approx(b, rel=1e-13)
    # single component, kappa = 2, at its mode
    one = np.zeros(1, dtype=abi.MIXTURE_DTYPE)
    one["k"], one["dim"], one["c"] = 1, 3, 1.0
    one["mu"][0, 0] = [0.0, 0.0, 1.0]
    one["kappa"][0, 0], one["lambda"][0, 0] = 2.0, 1.0
    peak = ref.fn("mixture_pdf")(abi.vptr(one), abi.ptr(np.array([0.0, 0.0, 1.0])))
    # proj/tests/test_sphdist.cpp:91-95: 2 e^2 / (4 pi sinh 2) to 1e-12 (the
    # literal 0.324236 there is checked with doctest's loose epsilon)
    assert peak == pytest.approx(2.0 * math.exp(2.0) / (4.0 * math.pi * math.sinh(2.0)), rel=1e-12)
    assert orc.fn("mixture_pdf")(abi.vptr(one), abi.ptr(np.array([0.0, 0.0, 1.0]))) == pytest.approx(peak, rel=1e-14)
    # gradient through a 2D-position field with a d = 3 mixture
    pr = make_preset("neumann-strip-vlin")
    cfg = abi.field_config(mixture_dim=3)
    fo, fr = orc.field(cfg, pr.scene.bbox, 5), ref.field(cfg, pr.scene.bbox, 5)
    recs = np.zeros(300, dtype=abi.GUIDE_RECORD_DTYPE)
    recs["x"] = rng.uniform(0.02, 0.98, (300, 2))
    nu = rng.normal(size=(300, 3))
    recs["nu"] = nu / np.linalg.norm(nu, axis=1)[:, None]
    recs["target"] = rng.uniform(0.0, 2.0, 300)
    recs["pdf_mis"] = rng.uniform(0.05, 0.5, 300)
    recs["pdf_g"] = rng.uniform(0.05, 0.5, 300)
    recs["pdf_u"] = 1.0 / (4.0 * np.pi)
    recs["c"] = 0.5
    recs["on_neumann"] = rng.integers(0, 2, 300)
    recs["normal"] = np.where(rng.random((300, 1)) < 0.5, [[0.0, 1.0]], [[0.0, -1.0]])
    tc = abi.train_config()
    go, gr = orc.field_grad(fo, recs, tc), ref.field_grad(fr, recs, tc)
    np.testing.assert_allclose(go, gr, rtol=1e-9, atol=1e-14 * np.abs(gr).max())
