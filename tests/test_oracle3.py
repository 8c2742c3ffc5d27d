"""The 3D oracle (oracle/wost3d.inc) on CPU: closed forms on the box domain,
brute force on random triangle soups, silhouette classification, the 3D
field's interpolation properties, and walk statistics against the analytic
solution. There is no reference 3D code, so these checks are what pins the
3D contract ("parity unpinned" against the reference; the d = 3 vMF pieces
it uses are pinned in tests/test_oracle.py)."""
import math

import numpy as np
import pytest

from fixtures3 import brute_closest, brute_ray, directions3, jittered_box, probes3, soup_scene
from oracle_lib import Oracle3
from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.scene3 import make_preset3, slice_points, strip_vlin_np


@pytest.fixture(scope="module")
def o3():
    return Oracle3()


def test_box_closed_forms(o3):
    p = make_preset3("box-strip-vlin", n=8)
    h = o3.scene(p.scene)
    x = probes3(1, 3000, 0.01, 0.99)
    _, d, tri = o3.closest_point(h, x, abi.KIND_DIRICHLET)
    assert np.array_equal(d, np.minimum(x[:, 0], 1 - x[:, 0]))
    # the silhouette of the insulated lateral faces = perimeters of the x faces
    ds = o3.closest_silhouette(h, x)
    lat = np.minimum.reduce([x[:, 1], 1 - x[:, 1], x[:, 2], 1 - x[:, 2]])
    np.testing.assert_allclose(ds, np.hypot(np.minimum(x[:, 0], 1 - x[:, 0]), lat), rtol=1e-15)
    dirs = directions3(2, 3000)
    t, hp, nrm, tri, kind = o3.ray_first_hit(h, x, dirs, 10.0, abi.KIND_ALL)
    with np.errstate(divide="ignore"):
        tt = np.min([np.where(dirs[:, a] > 0, (1 - x[:, a]) / dirs[:, a], -x[:, a] / dirs[:, a])
                     for a in range(3)], axis=0)
    np.testing.assert_allclose(t, tt, rtol=1e-13)
    assert (np.sum(nrm * dirs, axis=1) < 0).all()  # normals face the incoming ray
    np.testing.assert_allclose(np.linalg.norm(nrm, axis=1), 1.0, rtol=1e-15)
    # t_max cut and exclude
    t2, *_ = o3.ray_first_hit(h, x, dirs, tt * 0.5, abi.KIND_ALL)
    assert np.isinf(t2).all()
    r = o3.star_radius(h, x, 1e-3)
    assert (r <= d + 0.0).all()
    # x-face perimeters are always silhouettes; the lateral creases are convex
    # from the domain and dropped
    assert o3.silhouette_info(h) == (8 * 8, 0)
    o3.scene_destroy(h)


def test_obstacle_silhouette_counts(o3):
    p = make_preset3("box-strip-vlin-obstacle", n=8)
    h = o3.scene(p.scene)
    # obstacle_n = 4: its 12 edges x 4 segments are reflex creases (kept);
    # the box's lateral creases are convex (dropped)
    assert o3.silhouette_info(h) == (8 * 8, 12 * 4)
    # a point facing one obstacle face sees its rim edges: silhouette within
    # reach; a point far away in the corner of the box does too (box creases
    # never flip from inside, the obstacle's do)
    x = np.array([[0.5, 0.5, 0.15], [0.1, 0.1, 0.9]])
    ds = o3.closest_silhouette(h, x)
    assert ds[0] < 0.5 and np.isfinite(ds).all()
    o3.scene_destroy(h)


@pytest.mark.parametrize("seed", [1, 2])
def test_soup_bvh_matches_brute_force(o3, seed):
    sc = soup_scene(seed, 400)
    h = o3.scene(sc)
    x = probes3(seed + 10, 200)
    for kinds, sel in [(abi.KIND_ALL, np.ones(sc.n_tris, bool)), (abi.KIND_DIRICHLET, sc.kind == 0),
                       (abi.KIND_NEUMANN, sc.kind == 1)]:
        _, d, tri = o3.closest_point(h, x, kinds)
        bf = brute_closest(sc.tris[sel], x)
        ids = np.flatnonzero(sel)
        np.testing.assert_allclose(d, np.sqrt(bf.min(axis=1)), rtol=1e-12, atol=1e-15)
        best = ids[np.argmin(bf, axis=1)]
        gap = np.sort(bf, axis=1)
        clear = (gap[:, 1] - gap[:, 0]) > 1e-12
        assert np.array_equal(tri[clear], best[clear])
    dirs = directions3(seed + 20, 200)
    t, *_ = o3.ray_first_hit(h, x, dirs, 2.0, abi.KIND_ALL)
    tb = brute_ray(sc.tris, x, dirs, o3.fn("t_epsilon")(h), 2.0)
    np.testing.assert_allclose(t, tb, rtol=1e-12)
    o3.scene_destroy(h)


def test_jittered_box_creases_and_scene_errors(o3):
    sc = jittered_box(3, n=6)
    h = o3.scene(sc)
    a, c = o3.silhouette_info(h)
    assert c > 50  # jitter turns shared lateral edges into creases, about half of them reflex
    x = probes3(4, 500, 0.1, 0.9)
    ds = o3.closest_silhouette(h, x)
    assert np.isfinite(ds).all()
    o3.scene_destroy(h)
    bad = make_preset3("box-strip-vlin", n=2).scene
    bad.tris = bad.tris.copy()
    bad.tris[0, 1] = bad.tris[0, 0]  # degenerate
    with pytest.raises(Exception):
        o3.scene(bad)


def test_field3_init_and_interpolation(o3):
    cfg = abi.field_config3()
    f = o3.field(cfg, (0, 0, 0, 1, 1, 1), 7)
    p = o3.field_params(f)
    assert len(p) == abi.field_param_count3(cfg)
    emb = sum(r ** 3 * 4 for r in (8, 16, 32, 64))
    assert np.abs(p[:emb]).max() <= 1e-4
    x = probes3(5, 64)
    out = o3.field_eval(f, x, 41)
    assert out.shape == (64, 41) and np.isfinite(out).all()
    # partition of unity: a constant grid gives that constant input everywhere
    q = p.copy()
    q[:emb] = 0.25
    o3.field_set_params(f, q)
    a = o3.field_eval(f, x, 41)
    b = o3.field_eval(f, probes3(6, 64), 41)
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)
    o3.field_destroy(f)


def test_uniform_walks_match_analytic(o3):
    """Box domain, uniform 3D WoSt: per-point means within 4 SE of the
    strip_vlin series (the 3D solution is z-independent)."""
    p = make_preset3("box-strip-vlin", n=8)
    h = o3.scene(p.scene)
    x = slice_points(6, 6)
    st = o3.run(h, None, abi.solver_config("uniform"), x, 1, 400)
    ref = strip_vlin_np(x[:, 0], x[:, 1])
    se = np.sqrt(st["m2"] / (st["count"] - 1) / st["count"])
    z = (st["mean"] - ref) / np.maximum(se, 1e-12)
    assert np.abs(z).max() < 4.5, z
    assert abs(z.mean()) < 4.0 / math.sqrt(len(z)) * 1.5
    o3.scene_destroy(h)


def test_guided_walk_records(o3):
    """Guided walks write one record per step; targets follow the backward
    product (target_k = |g * prod_{j>k} mult_j| with rr = 1 below depth 128)."""
    p = make_preset3("box-strip-vlin", n=4)
    h = o3.scene(p.scene)
    f = o3.field(abi.field_config3(), (0, 0, 0, 1, 1, 1), 3)
    cfg = abi.solver_config("learnable_mis")
    x = slice_points(4, 4)
    recs = o3.walk_records(h, f, cfg, x, 9, 0)
    est, esc, steps = o3.walks(h, f, cfg, x, 9, 0)
    assert len(recs) == steps[esc == 0].sum()
    np.testing.assert_allclose(np.linalg.norm(recs["nu"], axis=1), 1.0, rtol=1e-12)
    pm = recs["c"] * recs["pdf_g"] + (1 - recs["c"]) * recs["pdf_u"]
    np.testing.assert_allclose(recs["pdf_mis"], pm, rtol=1e-12)
    assert (recs["target"] >= 0).all()
    o3.field_destroy(f)
    o3.scene_destroy(h)


def test_silhouette_index_equals_raw_facing_rule(o3):
    """Dropping coplanar and domain-convex creases from the index leaves the
    closest silhouette of every interior point unchanged: a numpy brute force
    over ALL Neumann edges with the plain facing rule (open edges always,
    shared edges when n0.(a-x) and n1.(a-x) differ in sign) agrees."""
    sc = jittered_box(9, n=5)
    h = o3.scene(sc)
    x = probes3(10, 300, 0.08, 0.92)
    got = o3.closest_silhouette(h, x)
    edges = {}
    for t, k in zip(sc.tris, sc.kind):
        if k != abi.NEUMANN:
            continue
        n = np.cross(t[1] - t[0], t[2] - t[0])
        n /= np.linalg.norm(n)
        for i in range(3):
            p, q = t[i], t[(i + 1) % 3]
            key = tuple(sorted((tuple(p), tuple(q))))
            edges.setdefault(key, []).append(n)
    want = np.full(len(x), np.inf)
    for (p, q), ns in edges.items():
        p, q = np.array(p), np.array(q)
        ab = q - p
        s = np.clip(((x - p) @ ab) / (ab @ ab), 0.0, 1.0)
        d = np.linalg.norm(x - (p + s[:, None] * ab), axis=1)
        if len(ns) == 2:
            f0, f1 = (p - x) @ ns[0], (p - x) @ ns[1]
            sil = f0 * f1 <= 0.0
        else:
            sil = np.ones(len(x), bool)
        want = np.where(sil, np.minimum(want, d), want)
    np.testing.assert_allclose(got, want, rtol=1e-12)
    o3.scene_destroy(h)


def test_source_term_matches_analytic(o3):
    """The d = 3 source term (Green's mass R^2/6, d = 3 radius CDF) against
    u = x^2 with f = 2 (Delta u = f, the reference's sign)."""
    p = make_preset3("box-poisson", n=6)
    h = o3.scene(p.scene)
    x = slice_points(5, 5)
    st = o3.run(h, None, abi.solver_config("uniform"), x, 3, 600)
    ref = np.array([p.analytic(*q) for q in x])
    se = np.sqrt(st["m2"] / (st["count"] - 1) / st["count"])
    z = (st["mean"] - ref) / np.maximum(se, 1e-12)
    assert np.abs(z).max() < 4.5, z
    assert abs(z.mean()) < 1.5
    o3.scene_destroy(h)


def test_flux_term_direction(o3):
    """The d = 3 Neumann-flux term is the reference's direction-sampled
    estimator (wost.cpp:89-109) with 4 pi t^2: it samples G h over the Neumann
    boundary a ray from x reaches, so a walker sitting on a flux face never
    samples that face (grazing directions, measure zero) - the 2D reference
    has the same property and no preset with h != 0. On u = y it moves the
    estimate from the zero-flux solution towards y (not all the way)."""
    p0 = make_preset3("box-flux", n=6)
    p0.scene.values[2] = (0, 0.0, 0.0, 0.0, 0.0)
    p0.scene.values[3] = (0, 0.0, 0.0, 0.0, 0.0)
    p1 = make_preset3("box-flux", n=6)
    x = slice_points(5, 5)
    means = []
    for p in (p0, p1):
        h = o3.scene(p.scene)
        means.append(o3.run(h, None, abi.solver_config("uniform"), x, 3, 400)["mean"].reshape(5, 5).mean(axis=1))
        o3.scene_destroy(h)
    ref = np.array([0.1, 0.3, 0.5, 0.7, 0.9])
    no_flux, flux = means
    assert abs(flux[0] - ref[0]) < abs(no_flux[0] - ref[0]) and abs(flux[4] - ref[4]) < abs(no_flux[4] - ref[4])
