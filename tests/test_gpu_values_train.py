"""GPU parity against the reference itself (oracle/_ref, the unmodified
proj/src compiled by oracle/Makefile) on paths the presets never exercise:

* Neumann flux h != 0 in 2D: sample_neumann_contrib (proj/src/wost.cpp:89-109,
  call site :198-203), per walk on the bit-faithful path and statistically on
  the tensor-core product path;
* raster boundary values and a raster source (RasterGrid::at,
  proj/src/scene.cpp:13-20; eval_source :53-67) on the device;
* one Adam step on a fixed gradient (GuidingField::adam_step,
  proj/src/guide_field.cpp:317-331);
* train_batch accounting on identical host records (proj/src/guide_train.cpp:94-198).
"""
import numpy as np
import pytest

from paper_2410_18944_b200 import abi, api
from fixtures import BOX, flux_scene, raster_scene
from paper_2410_18944_b200.scene import cell_centers, make_preset

pytestmark = pytest.mark.gpu


def _exact_walks(scene, field_g, mode, xy, seed, wpp):
    s = api.Solver(api.Accel(scene), field_g, abi.solver_config(mode), api.MLP_EXACT)
    s.set_points(xy)
    s.solve_rounds(seed, wpp, 1)
    return s.walks()


def _ref_field(ref, cfg, bbox, seed):
    return ref.field(cfg, bbox, seed)


@pytest.mark.parametrize("mode", ["uniform", "learnable_mis"])
@pytest.mark.parametrize("which", ["flux", "raster"])
def test_exact_walks_match_reference_per_walk(gpu, ref, which, mode):
    """Same PCG32 stream per walk, fp64 walk arithmetic in the reference's
    order: per-walk estimates agree to 1e-9 for >= 99% of walks (guided: the
    reference's fp32 MLP bit for bit), escapes agree."""
    scene = flux_scene() if which == "flux" else raster_scene()
    xy = cell_centers(48, 48, (0.02, 0.02, 0.98, 0.98))
    if which == "raster":  # inside the 24-gon
        xy = xy[np.hypot(xy[:, 0] - 0.5, xy[:, 1] - 0.5) < 0.42]
    h = ref.scene(scene)
    if which == "flux":
        assert ref.fn("has_neumann_flux")(h) == 1
    fo = fg = None
    if mode != "uniform":
        cfg = abi.field_config()
        fo = _ref_field(ref, cfg, scene.bbox, 17)
        fg = api.GuidingField(cfg, scene.bbox, 17)
        assert np.array_equal(ref.field_params(fo), fg.params())
    for wpp in (0, 3):
        est_r, esc_r, _ = ref.walks(h, fo, abi.solver_config(mode), xy, 11, wpp)
        est_g, esc_g, _ = _exact_walks(scene, fg, mode, xy, 11, wpp)
        close = np.abs(est_r - est_g) <= 1e-9 * np.maximum(1.0, np.abs(est_r))
        assert close.mean() >= 0.99, close.mean()
        assert (esc_r == esc_g).mean() >= 0.999
        # the flux / source terms contribute: estimates are not the g-only ones
        assert np.std(est_r) > 0


def test_flux_tensor_path_matches_reference_statistically(gpu, ref):
    """The product path (tcgen05 MLP, fp32 mixture, online training) on the
    flux scene against the reference's uniform solve of the same points:
    per-point means within 3 combined standard errors (<= 2% outliers), mean
    z centred."""
    scene = flux_scene()
    xy = cell_centers(24, 24, (0.05, 0.05, 0.95, 0.95))
    h = ref.scene(scene)
    st_r = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
    for w in range(128):
        ref.solve_batch(h, None, abi.solver_config("uniform"), xy, st_r, 3, w)
    f = api.GuidingField(abi.field_config(), scene.bbox, 3)
    s = api.Solver(api.Accel(scene), f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(xy)
    s.run(3, 256, 64, abi.train_config(seed=3))
    st_g = s.stats()
    se = np.sqrt(st_r["m2"] / (st_r["count"] * (st_r["count"] - 1)) +
                 st_g["m2"] / (st_g["count"] * (st_g["count"] - 1)))
    z = (st_g["mean"] - st_r["mean"]) / se
    assert np.mean(np.abs(z) > 3.0) <= 0.02, np.mean(np.abs(z) > 3.0)
    assert abs(z.mean()) < 4.0 / np.sqrt(len(z)), z.mean()


def test_raster_tensor_path_matches_reference_statistically(gpu, ref):
    scene = raster_scene()
    xy = cell_centers(24, 24, (0.1, 0.1, 0.9, 0.9))
    xy = xy[np.hypot(xy[:, 0] - 0.5, xy[:, 1] - 0.5) < 0.4]
    h = ref.scene(scene)
    st_r = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
    for w in range(128):
        ref.solve_batch(h, None, abi.solver_config("uniform"), xy, st_r, 4, w)
    f = api.GuidingField(abi.field_config(), scene.bbox, 4)
    s = api.Solver(api.Accel(scene), f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(xy)
    s.run(4, 256, 64, abi.train_config(seed=4))
    st_g = s.stats()
    se = np.sqrt(st_r["m2"] / (st_r["count"] * (st_r["count"] - 1)) +
                 st_g["m2"] / (st_g["count"] * (st_g["count"] - 1)))
    z = (st_g["mean"] - st_r["mean"]) / se
    assert np.mean(np.abs(z) > 3.0) <= 0.02, np.mean(np.abs(z) > 3.0)
    assert abs(z.mean()) < 4.0 / np.sqrt(len(z)), z.mean()


def test_adam_steps_match_reference(gpu, ref):
    """Three Adam steps on fixed gradients (the same fp32-representable values
    on both sides): parameters bit-equal to GuidingField::adam_step's for
    >= 99.99% of the 94,433, the rest within one fp32 ulp (device pow /
    glibc pow may differ in the last bit of the bias corrections)."""
    cfg = abi.field_config()
    fo = ref.field(cfg, BOX, 21)
    fg = api.GuidingField(cfg, BOX, 21)
    n = fg.n_params
    s = api.Solver(api.Accel(make_preset("neumann-strip").scene), fg, abi.solver_config("learnable_mis"))
    tc = abi.train_config(seed=1)
    rng = np.random.default_rng(8)
    for step in range(3):
        g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 0, n)).astype(np.float32)
        g[rng.random(n) < 0.05] = 0.0
        g64 = g.astype(np.float64)
        ref.lib.ref_field_adam_step(fo, abi.ptr(g64), tc.lr, tc.beta1, tc.beta2, tc.eps)
        buf = np.zeros(n + 1, dtype=np.float32)
        buf[:n] = g
        buf[n] = tc.minibatch  # record count = minibatch: the mean is the buffer itself
        s.train_apply(tc, buf)
    pr, pg = ref.field_params(fo), fg.params()
    assert fg.state()[3] == ref.lib.ref_field_adam_steps(fo) == 3
    eq = pr == pg
    assert eq.mean() >= 0.9999, eq.mean()
    ulp = np.abs(pr.view(np.int32).astype(np.int64) - pg.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1, ulp.max()


@pytest.mark.parametrize("cap,mb", [(1 << 15, 1 << 14), (3000, 1024)])
def test_train_batch_accounting_matches_reference(gpu, ref, cap, mb):
    """wostgpu_train_batch on the reference's own records: the reference's
    Fisher-Yates selection, so records seen / consumed / skipped (pdf floor,
    V floor) and Adam steps equal train_batch's; the trained parameters agree
    up to fp32-vs-fp64 gradient accumulation."""
    p = make_preset("neumann-strip-vlin")
    cfg = abi.field_config()
    h = ref.scene(p.scene)
    fo = ref.field(cfg, p.scene.bbox, 5)
    xy = cell_centers(32, 32, p.eval_bbox)
    st = np.zeros(len(xy), dtype=abi.POINT_STATS_DTYPE)
    recs = ref.solve_batch(h, fo, abi.solver_config("learnable_mis"), xy, st, 5, 0, collect=True)
    recs = recs.copy()
    recs["pdf_mis"][::97] = 1e-12  # below the pdf floor: skipped
    tc = abi.train_config(seed=9, max_records=cap, minibatch=mb)
    fg = api.GuidingField(cfg, p.scene.bbox, 5)
    p0 = fg.params().astype(np.float64)
    assert np.array_equal(ref.field_params(fo), fg.params())
    s = api.Solver(api.Accel(p.scene), fg, abi.solver_config("learnable_mis"))
    for rnd in (0, 1):
        sr = ref.train_batch(fo, recs, tc, rnd)
        sg = s.train_batch(recs, tc, rnd)
        for k in ("records_seen", "records_consumed", "skipped_low_pdf", "skipped_low_v", "steps"):
            assert getattr(sg, k) == getattr(sr, k), (k, getattr(sg, k), getattr(sr, k))
        assert sr.steps == -(-min(len(recs) - sr.skipped_low_pdf, cap) // mb)
        np.testing.assert_allclose(sg.mean_grad_norm, sr.mean_grad_norm, rtol=1e-3)
    # Adam moves each parameter by ~lr * sign(mean gradient); fp32 vs fp64
    # sums flip signs only for gradients near 0: the updates agree in
    # direction and for almost every parameter. (The device sums with fp32
    # atomics in a run-dependent order, so which near-zero gradients flip
    # varies from run to run: the bounds leave room for that.)
    du_r = ref.field_params(fo).astype(np.float64) - p0
    du_g = fg.params().astype(np.float64) - p0
    cos = du_r @ du_g / (np.linalg.norm(du_r) * np.linalg.norm(du_g))
    d = np.abs(du_r - du_g)
    assert cos > 0.98, cos
    assert np.median(d) < 1e-3 * tc.lr and np.mean(d > 0.1 * tc.lr) < 0.06, (np.median(d), np.mean(d > 0.1 * tc.lr))


def test_field_backward_adam_and_param_access_match_reference(gpu, ref):
    """GuidingField facade entries against the reference's own methods:
    eval_with_tape + backward (guide_field.cpp:223-315) summed over points
    (fp64; the device sums points in another order), adam_step on that fp64
    gradient (guide_field.cpp:317-331), get_param / set_param."""
    cfg = abi.field_config()
    fo = ref.field(cfg, BOX, 31)
    fg = api.GuidingField(cfg, BOX, 31)
    rng = np.random.default_rng(2)
    xy = np.ascontiguousarray(rng.uniform(-0.1, 1.1, (300, 2)))
    d_out = np.ascontiguousarray(rng.standard_normal((300, fg.output_dim)))
    gr = np.zeros(fg.n_params)
    ref.lib.ref_field_backward(fo, len(xy), abi.ptr(xy), abi.ptr(d_out), abi.ptr(gr))
    gg = fg.backward(xy, d_out)
    assert np.count_nonzero(gr) > 1000
    np.testing.assert_allclose(gg, gr, rtol=1e-12, atol=1e-13 * np.abs(gr).max())
    g1, g2 = gr.copy(), gr.copy()
    ref.lib.ref_field_adam_step(fo, abi.ptr(g1), 1e-2, 0.9, 0.99, 1e-8)
    fg.adam_step(g2, 1e-2, 0.9, 0.99, 1e-8)
    assert not g2.any()  # zeroed, as the reference leaves it
    pr, pg = ref.field_params(fo), fg.params()
    assert (pr == pg).mean() >= 0.9999
    ulp = np.abs(pr.view(np.int32).astype(np.int64) - pg.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    fg.set_param(fg.n_params - 1, 0.25)
    assert fg.get_param(fg.n_params - 1) == 0.25 and fg.params()[-1] == np.float32(0.25)
