"""Estimator-level parity with the reference on cfg 2 (neumann-strip-vlin
128^2, 256 wpp, seed 1) against the reference's own per-point statistics
(tests/golden/ref_cfg2_*_seed1.npz, from its run_solve) and its relMSE over
seeds 1-8 (tests/golden/ref_cfg2_seeds.json, tests/golden/make_cfg2_seeds.py):
  * uniform WoSt: per-point means equal the reference's to 1e-9 (same PCG32
    streams, fp64 arithmetic in the same order);
  * learnable MIS with online training: per-point means within 3 combined
    standard errors for >= 99% of points, and the 8-seed mean relMSE and the
    variance-reduction factor over uniform within 10% of the reference's (a
    single seed's relMSE scatters by ~10%, dominated by a few rare
    high-throughput walks, so both sides average 8 seeds)."""
import json
import os

import numpy as np
import pytest

from paper_2410_18944_b200 import abi, api
from paper_2410_18944_b200.scene import cell_centers, make_preset, relmse

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _se(st):
    c = st["count"].astype(np.float64)
    return np.sqrt(st["m2"] / (c * (c - 1)))


def _run(mode, seed, mlp=api.MLP_TENSOR):
    pr = make_preset("neumann-strip-vlin")
    pts = cell_centers(128, 128, pr.eval_bbox)
    field = api.GuidingField(abi.field_config(), pr.scene.bbox, seed) if mode != "uniform" else None
    s = api.Solver(api.Accel(pr.scene), field, abi.solver_config(mode), mlp)
    s.set_points(pts)
    s.run(seed, 256, 256, abi.train_config(seed=seed) if field else None)
    ref = np.array([pr.analytic(x, y) for x, y in pts])
    return s.stats(), ref


def test_uniform_cfg1_identical_to_reference(gpu):
    st, ref = _run("uniform", 1)
    g = np.load(os.path.join(G, "ref_cfg2_uniform_seed1.npz"))
    # CUDA's fp64 exp/log/sin/cos are within 1-2 ulp of glibc's: per-point
    # means differ only at that level
    assert np.max(np.abs(st["mean"] - g["mean"])) < 1e-9
    assert int(st["escaped"].sum()) == int(g["escaped"].sum())
    assert relmse(st["mean"], ref) == pytest.approx(float(g["relmse"][0]), rel=1e-9)


@pytest.mark.parametrize("mlp", [api.MLP_TENSOR, api.MLP_EXACT])
def test_guided_cfg2_per_point_within_3_se(gpu, mlp):
    st, _ = _run("learnable_mis", 1, mlp)
    g = np.load(os.path.join(G, "ref_cfg2_learnable_seed1.npz"))
    s = np.sqrt(_se(st) ** 2 + g["se"] ** 2)
    frac = np.mean(np.abs(st["mean"] - g["mean"]) > 3.0 * s)
    assert frac < 0.01, frac
    # escapes stay at the reference's rate (t_eps pass-through, wost.cpp:259-263)
    assert int(st["escaped"].sum()) < 4 * int(g["escaped"].sum()) + 20


def test_guided_relmse_and_variance_reduction_within_10_percent(gpu):
    ref = json.load(open(os.path.join(G, "ref_cfg2_seeds.json")))
    ours_g, ours_u = [], []
    seeds = sorted(int(k) for k in ref["learnable_mis"])
    assert len(seeds) == 8
    for seed in seeds:
        st, img = _run("learnable_mis", seed)
        ours_g.append(relmse(st["mean"], img))
        st, img = _run("uniform", seed)
        ours_u.append(relmse(st["mean"], img))
    ref_g = np.mean(list(ref["learnable_mis"].values()))
    ref_u = np.mean(list(ref["uniform"].values()))
    assert abs(np.mean(ours_g) - ref_g) / ref_g < 0.10, (ours_g, ref_g)
    vr_ours, vr_ref = np.mean(ours_u) / np.mean(ours_g), ref_u / ref_g
    assert abs(vr_ours - vr_ref) / vr_ref < 0.10, (vr_ours, vr_ref)


def _trimmed(v, frac=0.1):
    """mean of the central 80% (one run in ~20 of the learned estimator has
    a few high-weight walks that lift its relMSE 2-10x, on the reference and
    here alike)"""
    v = np.sort(np.asarray(v, dtype=np.float64))
    k = int(round(len(v) * frac))
    return float(v[k:len(v) - k].mean())


@pytest.mark.parametrize("walk", ["wave", "lockstep"])
def test_cfg3_seeds_relmse_and_vr_within_10_percent(gpu, monkeypatch, walk):
    """cfg 3 (const-source-disk: source term f = 4, eps = 1e-6, learnable MIS
    trained every round) at 128^2 x 256 wpp over 64 seeds, through the 2D
    wavefront pair (forced: the pair the configured 512^2 grid selects) and
    the lockstep kernel (the default at 128^2), against the reference's own
    run_solve over its seeds (tests/golden/ref_cfg3_seeds.json,
    tests/golden/make_cfg3_seeds.py): the trimmed-mean relMSE and the
    variance-reduction factor over uniform within 10% of the reference's.
    Uniform walks are the reference's walk for walk (seed 1 checked), so
    both VR factors share the reference's uniform relMSE. Training sums
    gradients with fp32 atomics, so our per-seed relMSE varies from run to
    run: a 32-seed trimmed mean moved by 8% between two runs, 64 seeds bring
    its spread to ~3-4% (bootstrap over 64-seed runs: ratio 1.01 wave / 1.03
    lockstep against the reference's seeds)."""
    with open(os.path.join(G, "ref_cfg3_seeds.json")) as f:
        ref = json.load(f)
    ref_g = [float(v) for v in ref["learnable_mis"].values()]
    ref_u = float(np.mean([float(v) for v in ref["uniform"].values()]))
    assert len(ref_g) >= 15
    monkeypatch.setenv("WOSTGPU_WALK2", walk)
    pr = make_preset("const-source-disk")
    pts = cell_centers(128, 128, pr.eval_bbox)
    truth = np.array([pr.analytic(x, y) for x, y in pts])
    acc = api.Accel(pr.scene)
    g = []
    for seed in range(1, 65):
        f = api.GuidingField(abi.field_config(), pr.scene.bbox, seed)
        s = api.Solver(acc, f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
        s.set_points(pts)
        s.run(seed, 256, 256, abi.train_config(seed=seed))
        g.append(relmse(s.stats()["mean"], truth))
    us = api.Solver(acc, None, abi.solver_config("uniform"))
    us.set_points(pts)
    us.run(1, 256, 0, None)
    assert relmse(us.stats()["mean"], truth) == pytest.approx(float(ref["uniform"]["1"]), rel=1e-6)
    ours, theirs = _trimmed(g), _trimmed(ref_g)
    assert abs(ours / theirs - 1.0) < 0.10, (ours, theirs)
    assert abs((ref_u / ours) / (ref_u / theirs) - 1.0) < 0.10, (ref_u / ours, ref_u / theirs)


def test_cfg3_512_wavefront_per_point_matches_reference(gpu):
    """cfg 3 at its configured size (const-source-disk, 512^2 points, 256 wpp,
    learnable MIS trained every round, seed 1) through the product's 2D
    wavefront pair (wg_wave2.cu: 256 segments and 262,144 walks per round
    select it) against the reference's own run_solve on the same
    configuration (tests/golden/ref_cfg3_512_seed1.npz, from
    tests/golden/make_cfg3_512.py): per-point means within 3 combined
    standard errors for >= 99% of the points with the mean z centred, and
    the single-seed relMSE within 25% (one seed's relMSE scatters ~15%; the
    10% relMSE criterion is tested over seeds at 128^2)."""
    g = np.load(os.path.join(G, "ref_cfg3_512_seed1.npz"))
    pr = make_preset("const-source-disk")
    pts = cell_centers(512, 512, pr.eval_bbox)
    truth = np.array([pr.analytic(x, y) for x, y in pts])
    f = api.GuidingField(abi.field_config(), pr.scene.bbox, 1)
    s = api.Solver(api.Accel(pr.scene), f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
    s.set_points(pts)
    s.run(1, 256, 256, abi.train_config(seed=1))
    st = s.stats()
    se = np.sqrt(_se(st) ** 2 + g["se"].astype(np.float64) ** 2)
    z = (st["mean"] - g["mean"].astype(np.float64)) / se
    assert np.mean(np.abs(z) > 3.0) < 0.01, np.mean(np.abs(z) > 3.0)
    assert abs(z.mean()) < 4.0 / np.sqrt(len(z)), z.mean()
    rel = relmse(st["mean"], truth)
    assert abs(rel / float(g["relmse"][0]) - 1.0) < 0.25, (rel, float(g["relmse"][0]))
