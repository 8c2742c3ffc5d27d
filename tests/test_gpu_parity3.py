"""GPU parity of the 3D path (include/wostgpu3.h) against the 3D oracle
(oracle/wost3d.inc) on the same inputs: geometry bit for bit (fp64, same
operation order, order-independent selection rules), field initialisation
and exact evaluation bit for bit, per-walk estimates to 1e-9 for >= 99.9% /
99% of walks (uniform / guided; ulp-level libm differences only), records
and training gradients to the stated tolerances, and walk statistics
against the analytic solution of the box domain."""
import numpy as np
import pytest

from fixtures3 import directions3, jittered_box, probes3, soup_scene
from oracle_lib import Oracle3
from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.api3 import MLP_EXACT, MLP_TENSOR, Accel3, GuidingField3, Solver3
from paper_2410_18944_b200.scene3 import make_preset3, slice_points, strip_vlin_np

pytestmark = pytest.mark.gpu

BOX = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)


@pytest.fixture(scope="module")
def o3():
    return Oracle3()


def _scenes():
    return {
        "box": make_preset3("box-strip-vlin", n=16).scene,
        "obstacle": make_preset3("box-strip-vlin-obstacle", n=12).scene,
        "soup": soup_scene(11, 3000),
        "jitter": jittered_box(5, n=10),
    }


@pytest.mark.parametrize("name", ["box", "obstacle", "soup", "jitter"])
def test_geometry_bit_exact(gpu, o3, name):
    sc = _scenes()[name]
    ho, acc = o3.scene(sc), Accel3(sc)
    info = acc.info()
    assert (info["sil_always"], info["sil_crease"]) == o3.silhouette_info(ho)
    assert info["t_epsilon"] == o3.fn("t_epsilon")(ho)
    x = probes3(21, 4000, 0.005, 0.995)
    for kinds in (abi.KIND_DIRICHLET, abi.KIND_NEUMANN, abi.KIND_ALL):
        a, b = o3.closest_point(ho, x, kinds), acc.closest_point(x, kinds)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    assert np.array_equal(o3.closest_silhouette(ho, x), acc.closest_silhouette(x))
    d = directions3(22, 4000)
    tmax = np.random.default_rng(3).uniform(0.05, 1.5, 4000)
    ex = np.random.default_rng(4).integers(-1, sc.n_tris, 4000).astype(np.int32)
    for kinds in (abi.KIND_NEUMANN, abi.KIND_ALL):
        a = o3.ray_first_hit(ho, x, d, tmax, kinds, ex)
        b = acc.ray_first_hit(x, d, tmax, kinds, ex)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    if name != "soup":  # soups may leave star regions unbounded
        assert np.array_equal(o3.star_radius(ho, x, 1e-3), acc.star_radius(x, 1e-3))
    o3.scene_destroy(ho)


def test_too_deep_tree_falls_back_to_median_splits(gpu, o3, capfd, monkeypatch):
    """The scene build checks each 4-wide tree against the device traversal
    stacks (3 x depth entries): a surface-area-split tree that does not fit
    is rebuilt with median splits (WOSTGPU_BVH3_STATS prints both attempts)
    and answers every query exactly like the oracle; a scene whose median
    tree does not fit either is rejected with WG_ERR_INVALID. The capacity
    is lowered through the WOSTGPU_BVH3_STACK test hook."""
    sc = soup_scene(13, 3000)
    sc.kind[:] = abi.DIRICHLET  # one tree (no Neumann / silhouette-edge trees)
    sc.value_index[:] = 1
    monkeypatch.setenv("WOSTGPU_BVH3_STATS", "1")
    capfd.readouterr()
    Accel3(sc)
    depths = [int(ln.rsplit("depth", 1)[1]) for ln in capfd.readouterr().err.splitlines()
              if ln.startswith("bvh3 dirichlet")]
    assert len(depths) == 1, depths
    monkeypatch.setenv("WOSTGPU_BVH3_STACK", str(3 * depths[0] - 1))  # the SAH tree no longer fits
    acc = Accel3(sc)
    lines = [ln for ln in capfd.readouterr().err.splitlines() if ln.startswith("bvh3 dirichlet")]
    assert len(lines) == 2, lines  # the SAH attempt, then the median rebuild
    assert int(lines[1].rsplit("depth", 1)[1]) < depths[0]
    ho = o3.scene(sc)
    x = probes3(23, 3000, 0.0, 1.0)
    for kinds in (abi.KIND_DIRICHLET, abi.KIND_ALL):
        a, b = o3.closest_point(ho, x, kinds), acc.closest_point(x, kinds)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    d = directions3(24, 3000)
    tmax = np.full(3000, 2.0)
    ex = np.full(3000, -1, dtype=np.int32)
    a = o3.ray_first_hit(ho, x, d, tmax, abi.KIND_ALL, ex)
    b = acc.ray_first_hit(x, d, tmax, abi.KIND_ALL, ex)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    o3.scene_destroy(ho)
    monkeypatch.setenv("WOSTGPU_BVH3_STACK", "3")  # not even a median tree fits
    with pytest.raises(Exception, match="too deep"):
        Accel3(sc)


def test_field3_init_and_eval_bit_exact(gpu, o3):
    cfg = abi.field_config3()
    fo = o3.field(cfg, BOX, 13)
    fg = GuidingField3(cfg, BOX, 13)
    assert np.array_equal(o3.field_params(fo), fg.params())
    x = np.concatenate([probes3(1, 3000, -0.1, 1.1), np.array([[0, 0, 0], [1, 1, 1], [0.5, 1.0, 0.0]])])
    assert np.array_equal(o3.field_eval(fo, x, 41), fg.eval_batch(x))
    # after a parameter change (set_state path)
    p = fg.params() + np.float32(0.01) * np.random.default_rng(2).standard_normal(fg.n_params).astype(np.float32)
    fg.set_params(p)
    o3.field_set_params(fo, p)
    assert np.array_equal(o3.field_eval(fo, x, 41), fg.eval_batch(x))
    o3.field_destroy(fo)


def _outside_obstacle(x):
    """Evaluation points of the obstacle scene must lie in the domain: a walk
    started inside the insulated obstacle never meets a Dirichlet boundary."""
    inside = ((x[:, 0] > 0.35) & (x[:, 0] < 0.65) & (x[:, 1] > 0.35) & (x[:, 1] < 0.65) &
              (x[:, 2] > 0.3) & (x[:, 2] < 0.7))
    return x[~inside]


def _walks(o3, sc, cfg, x, seed, field_o=None, field_g=None):
    ho = o3.scene(sc)
    est_o, esc_o, steps_o = o3.walks(ho, field_o, cfg, x, seed, 0)
    sol = Solver3(Accel3(sc), field_g, cfg, MLP_EXACT)
    sol.set_points(x)
    sol.solve_rounds(seed, 0, 1)
    est_g, esc_g, steps_g = sol.walks()
    o3.scene_destroy(ho)
    return est_o, esc_o, steps_o, est_g, esc_g, steps_g


@pytest.mark.parametrize("name", ["box", "obstacle", "jitter"])
def test_uniform_walks_match_oracle_per_walk(gpu, o3, name):
    sc = _scenes()[name]
    x = _outside_obstacle(probes3(31, 3000, 0.05, 0.95))
    est_o, esc_o, st_o, est_g, esc_g, st_g = _walks(o3, sc, abi.solver_config("uniform"), x, 7)
    close = np.abs(est_o - est_g) <= 1e-9 * np.maximum(1.0, np.abs(est_o))
    assert close.mean() >= 0.999, close.mean()
    assert (st_o == st_g).mean() >= 0.999
    assert (esc_o == esc_g).mean() >= 0.999


@pytest.mark.parametrize("mode", ["guiding_only", "fixed_mis", "learnable_mis"])
def test_guided_walks_exact_mlp_match_oracle(gpu, o3, mode):
    sc = _scenes()["obstacle"]
    cfg_f = abi.field_config3()
    fo, fg = o3.field(cfg_f, BOX, 17), GuidingField3(cfg_f, BOX, 17)
    # a non-trivial field: random perturbation of the initial parameters
    p = fg.params()
    p = p + np.float32(0.3) * np.random.default_rng(8).standard_normal(len(p)).astype(np.float32)
    fg.set_params(p)
    o3.field_set_params(fo, p)
    x = _outside_obstacle(probes3(41, 1500, 0.05, 0.95))
    est_o, esc_o, st_o, est_g, esc_g, st_g = _walks(o3, sc, abi.solver_config(mode), x, 99, fo, fg)
    close = np.abs(est_o - est_g) <= 1e-9 * np.maximum(1.0, np.abs(est_o))
    assert close.mean() >= 0.99, close.mean()
    o3.field_destroy(fo)


def test_records_match_oracle(gpu, o3):
    """A collecting round writes the oracle's records (one per step of every
    finished walk) with the same pdfs and backward-product targets."""
    sc = make_preset3("box-strip-vlin", n=8).scene
    cfg_f = abi.field_config3()
    fo, fg = o3.field(cfg_f, BOX, 23), GuidingField3(cfg_f, BOX, 23)
    cfg = abi.solver_config("learnable_mis")
    x = slice_points(24, 24)
    ho = o3.scene(sc)
    rec_o = o3.walk_records(ho, fo, cfg, x, 5, 0)
    sol = Solver3(Accel3(sc), fg, cfg, MLP_EXACT)
    sol.set_points(x)
    sol.solve_rounds(5, 0, 1, collect=True)
    rec_g = sol.records()
    assert abs(len(rec_g) - len(rec_o)) <= max(2, len(rec_o) // 500)
    for k in ("pdf_mis", "pdf_g", "pdf_u", "c"):
        np.testing.assert_allclose(np.sort(rec_g[k]), np.sort(rec_o[k]), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np.sort(rec_g["target"]), np.sort(rec_o["target"]), rtol=1e-4, atol=1e-6)
    o3.scene_destroy(ho)
    o3.field_destroy(fo)


@pytest.mark.parametrize("mlp", [MLP_EXACT, MLP_TENSOR])
def test_field_grad_matches_oracle(gpu, o3, mlp):
    """3D training tiles against the oracle's fp64 gradient of the same
    minibatch: the CUDA-core tile (fp32 MLP, fp64 loss; MLP_EXACT) and the
    tcgen05 tile (grad3_tc_kernel: split-fp16 forward / backward / weight
    gradients in TMEM, fp64 loss at the outputs; MLP_TENSOR)."""
    sc = make_preset3("box-strip-vlin-obstacle", n=8).scene
    cfg_f = abi.field_config3()
    fo, fg = o3.field(cfg_f, BOX, 29), GuidingField3(cfg_f, BOX, 29)
    cfg = abi.solver_config("learnable_mis")
    ho = o3.scene(sc)
    recs = o3.walk_records(ho, fo, cfg, _outside_obstacle(probes3(3, 600, 0.05, 0.95)), 3, 0)
    tc = abi.train_config()
    g_o = o3.field_grad(fo, recs, tc)
    sol = Solver3(Accel3(sc), fg, cfg, mlp)
    g_g = sol.field_grad(recs, tc)
    scale = np.abs(g_o).max()
    assert scale > 0
    np.testing.assert_allclose(g_g, g_o, rtol=0, atol=2e-3 * scale)
    # direction agreement on the MLP block and the grid block separately
    emb = abi.field_param_count3(cfg_f) - (16 * 64 + 64 + 64 * 64 + 64 + 64 * 41 + 41)
    for sl in (slice(0, emb), slice(emb, None)):
        cos = g_g[sl] @ g_o[sl] / (np.linalg.norm(g_g[sl]) * np.linalg.norm(g_o[sl]))
        assert cos > 0.999, cos
    o3.scene_destroy(ho)
    o3.field_destroy(fo)


def test_uniform_run_matches_analytic(gpu):
    """cfg-4 shape at reduced size: the box domain (n = 91, 99,372 triangles),
    a 32 x 32 slice, 256 walks per point: per-point means within 4.5 SE of
    the strip_vlin series."""
    p = make_preset3("box-strip-vlin")
    x = slice_points(32, 32)
    sol = Solver3(Accel3(p.scene), None, abi.solver_config("uniform"))
    sol.set_points(x)
    sol.run(1, 256, 0, None)
    st = sol.stats()
    ref = strip_vlin_np(x[:, 0], x[:, 1])
    se = np.sqrt(st["m2"] / (st["count"] - 1) / st["count"])
    # next to x = 0 most walks end on g = 0 and the estimator is strongly
    # skewed (few non-zero samples): the per-point z test uses the interior
    ok = (st["m2"] > 0) & (x[:, 0] > 0.1)
    z = (st["mean"][ok] - ref[ok]) / se[ok]
    assert np.abs(z).max() < 5.0
    assert (np.abs(z) > 3.0).mean() < 0.01
    assert abs(z.mean()) < 0.2


def test_guided_training_reduces_error(gpu):
    """Online learning on the box domain: a guided learnable-MIS run (training
    every round) is unbiased and its relMSE at equal walks is not worse than
    uniform's by more than noise; the field's Adam step count advances."""
    p = make_preset3("box-strip-vlin", n=32)
    x = slice_points(24, 24)
    ref = strip_vlin_np(x[:, 0], x[:, 1])
    u = Solver3(Accel3(p.scene), None, abi.solver_config("uniform"))
    u.set_points(x)
    u.run(3, 64, 0, None)
    su = u.stats()
    f = GuidingField3(abi.field_config3(), BOX, 3)
    g = Solver3(Accel3(p.scene), f, abi.solver_config("learnable_mis"))
    g.set_points(x)
    tst, _ = g.run(3, 64, 64, abi.train_config(seed=3))
    sg = g.stats()
    assert tst.steps >= 64 and tst.records_consumed > 0
    rel = lambda s: float(np.mean((s["mean"] - ref) ** 2 / (ref ** 2 + 1e-4)))
    ok = (sg["m2"] > 0) & (x[:, 0] > 0.1)
    z = (sg["mean"][ok] - ref[ok]) / np.sqrt(sg["m2"][ok] / (sg["count"][ok] - 1) / sg["count"][ok])
    assert abs(z.mean()) < 0.25
    assert rel(sg) < 1.5 * rel(su), (rel(sg), rel(su))


def test_field3_tensor_eval_matches_exact(gpu):
    """tcgen05 MLP (split-fp16 operands, fp32 accumulation) against the exact
    fp32 evaluation: 1e-4 of each row's scale (the 2D path's bound)."""
    cfg = abi.field_config3()
    f = GuidingField3(cfg, BOX, 41)
    p = f.params()
    p = p + np.float32(0.2) * np.random.default_rng(4).standard_normal(len(p)).astype(np.float32)
    f.set_params(p)
    x = probes3(7, 5000, -0.05, 1.05)
    a, b = f.eval_batch(x, MLP_EXACT), f.eval_batch(x, MLP_TENSOR)
    scale = np.maximum(np.abs(a).max(axis=1, keepdims=True), 1e-3)
    assert (np.abs(a - b) / scale).max() < 1e-4


@pytest.mark.parametrize("mode", ["learnable_mis", "guiding_only"])
def test_tensor_walks_match_exact_statistically(gpu, mode):
    """Guided walks with the tcgen05 MLP kernel against the exact kernel on
    the obstacle scene (reflection, creases): per-point means over 128 walks
    agree within 4.5 combined SE, and the mean z is centred."""
    sc = make_preset3("box-strip-vlin-obstacle", n=12).scene
    cfg_f = abi.field_config3()
    f = GuidingField3(cfg_f, BOX, 5)
    p = f.params()
    p = p + np.float32(0.3) * np.random.default_rng(6).standard_normal(len(p)).astype(np.float32)
    f.set_params(p)
    x = _outside_obstacle(probes3(8, 400, 0.08, 0.92))
    out = []
    for mlp in (MLP_EXACT, MLP_TENSOR):
        s = Solver3(Accel3(sc), f, abi.solver_config(mode), mlp)
        s.set_points(x)
        s.run(12, 128, 0, None)
        out.append(s.stats())
    a, b = out
    se = np.sqrt(a["m2"] / (a["count"] - 1) / a["count"] + b["m2"] / (b["count"] - 1) / b["count"])
    ok = se > 0
    z = (a["mean"][ok] - b["mean"][ok]) / se[ok]
    assert np.abs(z).max() < 4.5
    assert abs(z.mean()) < 4.0 / np.sqrt(ok.sum())


@pytest.mark.parametrize("name", ["box-poisson", "box-flux"])
def test_source_and_flux_walks_match_oracle(gpu, o3, name):
    """d = 3 source (Green's mass, radius CDF, occlusion ray) and Neumann-flux
    terms: per-walk estimates equal the oracle's (same draws, same order)."""
    sc = make_preset3(name, n=10).scene
    x = probes3(51, 2000, 0.05, 0.95)
    for mode in ("uniform",):
        est_o, esc_o, st_o, est_g, esc_g, st_g = _walks(o3, sc, abi.solver_config(mode), x, 3)
        close = np.abs(est_o - est_g) <= 1e-9 * np.maximum(1.0, np.abs(est_o))
        assert close.mean() >= 0.999, close.mean()


def test_source_term_record_targets_match_oracle(gpu, o3):
    """Records of a scene with a source term carry the walk's backward suffix
    sums (target_k = |S_{k+1} / Q_k|, S += local_k), like the oracle's
    backfill with local terms."""
    sc = make_preset3("box-poisson", n=8).scene
    cfg_f = abi.field_config3()
    fo, fg = o3.field(cfg_f, BOX, 31), GuidingField3(cfg_f, BOX, 31)
    cfg = abi.solver_config("learnable_mis")
    x = slice_points(20, 20)
    ho = o3.scene(sc)
    rec_o = o3.walk_records(ho, fo, cfg, x, 7, 0)
    sol = Solver3(Accel3(sc), fg, cfg, MLP_EXACT)
    sol.set_points(x)
    sol.solve_rounds(7, 0, 1, collect=True)
    rec_g = sol.records()
    assert abs(len(rec_g) - len(rec_o)) <= max(2, len(rec_o) // 500)
    np.testing.assert_allclose(np.sort(rec_g["target"]), np.sort(rec_o["target"]), rtol=1e-4, atol=1e-6)
    o3.scene_destroy(ho)
    o3.field_destroy(fo)


def test_poisson_tensor_path_matches_analytic(gpu):
    """box-poisson (u = x^2, f = 2) through the product path (guided,
    tensor-core wavefront, online training): per-point means within SE of x^2."""
    p = make_preset3("box-poisson", n=32)
    x = slice_points(24, 24)
    f = GuidingField3(abi.field_config3(), BOX, 9)
    s = Solver3(Accel3(p.scene), f, abi.solver_config("learnable_mis"))
    s.set_points(x)
    s.run(9, 96, 32, abi.train_config(seed=9))
    st = s.stats()
    ref = x[:, 0] ** 2
    ok = (st["m2"] > 0) & (x[:, 0] > 0.1)
    z = (st["mean"][ok] - ref[ok]) / np.sqrt(st["m2"][ok] / (st["count"][ok] - 1) / st["count"][ok])
    assert np.abs(z).max() < 5.0
    assert abs(z.mean()) < 0.3


def test_error_paths(gpu):
    """The 3D boundary's failure modes map to the reference's exception
    classes (SceneError / invalid_argument), like the 2D C-ABI."""
    from paper_2410_18944_b200._lib import InvalidArgument, SceneError, WostGpuError
    from paper_2410_18944_b200.scene3 import Scene3
    from paper_2410_18944_b200 import api
    empty = Scene3(np.zeros((0, 3, 3)), np.zeros(0, np.int32), np.zeros(0, np.int32),
                   [(0, 0.0, 0.0, 0.0, 0.0)])
    with pytest.raises(SceneError):
        Accel3(empty)
    bad = make_preset3("box-strip-vlin", n=2).scene
    bad.value_index = bad.value_index.copy()
    bad.value_index[0] = 7  # undefined value
    with pytest.raises(SceneError):
        Accel3(bad)
    with pytest.raises(InvalidArgument):
        GuidingField3(abi.field_config(mixture_dim=2), BOX, 1)  # 3D fields need a d = 3 mixture
    with pytest.raises(InvalidArgument):
        GuidingField3(abi.field_config3(), (0, 0, 0, 1, 0, 1), 1)  # empty bbox
    acc = Accel3(make_preset3("box-strip-vlin", n=4).scene)
    with pytest.raises(InvalidArgument):
        Solver3(acc, None, abi.solver_config("learnable_mis"))  # guided without a field
    f2 = api.GuidingField(abi.field_config(), (0, 0, 1, 1), 1)
    with pytest.raises(WostGpuError):
        Solver3(acc, f2, abi.solver_config("learnable_mis"))  # a 2D field
    s = Solver3(acc, None, abi.solver_config("uniform"))
    with pytest.raises(WostGpuError):
        s.set_points(np.zeros((0, 3)))
    # a Neumann-only closed box: no Dirichlet boundary, no silhouette -> unbounded star
    only_n = make_preset3("box-strip-vlin", n=2).scene
    only_n.kind = np.full(only_n.n_tris, abi.NEUMANN, dtype=np.int32)
    only_n.value_index = np.zeros(only_n.n_tris, dtype=np.int32)
    acc_n = Accel3(only_n)
    with pytest.raises(SceneError):
        acc_n.star_radius(np.array([[0.5, 0.5, 0.5]]), 1e-3)
    sn = Solver3(acc_n, None, abi.solver_config("uniform"))
    sn.set_points(np.array([[0.5, 0.5, 0.5]]))
    with pytest.raises(SceneError):
        sn.run(1, 1, 0, None)


def test_field3_checkpoint_round_trip(gpu, tmp_path):
    """A trained 3D field saved (WGF1 layout, magic WGF3) and loaded gives the
    same parameters, Adam state and evaluation."""
    p = make_preset3("box-strip-vlin", n=8)
    f = GuidingField3(abi.field_config3(), BOX, 4)
    s = Solver3(Accel3(p.scene), f, abi.solver_config("learnable_mis"))
    s.set_points(slice_points(16, 16))
    s.run(4, 3, 3, abi.train_config(seed=4))
    path = str(tmp_path / "field.wgf3")
    f.save(path)
    g = GuidingField3.load(path)
    a, b = f.state(), g.state()
    for u, v in zip(a[:3], b[:3]):
        assert np.array_equal(u, v)
    assert a[3] == b[3] and a[3] >= 3
    x = probes3(9, 500)
    assert np.array_equal(f.eval_batch(x), g.eval_batch(x))


@pytest.mark.parametrize("name", ["box-strip-vlin-obstacle", "box-strip-vlin"])
@pytest.mark.parametrize("collect", [False, True])
@pytest.mark.parametrize("tail", ["0", "3000", "65536"])
def test_wavefront_walks_equal_lockstep_per_walk(gpu, monkeypatch, name, collect, tail):
    """The wavefront pair (geometry pass + tensor-core direction pass)
    against the lockstep tensor-core kernel: the
    same PCG32 streams, the same tcgen05 MLP rows and the same exact
    geometry minima, so every walk's estimate, escape flag and step count
    is identical; with record collection the record counts match too. The
    drain hand-off (wave_tail_kernel) is off, mid-drain (3,000 walks left)
    and immediate (all 18k walks)."""
    monkeypatch.setenv("WOSTGPU_WAVE3_TAIL", tail)
    sc = make_preset3(name, n=24).scene
    f = GuidingField3(abi.field_config3(), BOX, 8)
    p = f.params() + np.float32(0.3) * np.random.default_rng(9).standard_normal(f.n_params).astype(np.float32)
    f.set_params(p)
    x = _outside_obstacle(probes3(21, 6000, 0.03, 0.97))
    out = []
    for mode in ("lockstep", "wave"):
        monkeypatch.setenv("WOSTGPU_WALK3", mode)
        s = Solver3(Accel3(sc), f, abi.solver_config("learnable_mis"), MLP_TENSOR)
        s.set_points(x)
        s.solve_rounds(4, 3, 1, collect=collect)
        out.append(s.walks() + ((len(s.records()),) if collect else (0,)))
    (ea, sa, na, ra), (eb, sb, nb, rb) = out
    assert np.array_equal(sa, sb) and np.array_equal(na, nb)
    assert np.array_equal(ea, eb)
    assert ra == rb and (ra > 0) == collect
