"""The reference's harness re-linked to the GPU path:
run_solve writes the reference's result files and convergence log,
run_ablation compares the sampler modes at equal samples, run_equal_time at
equal wall time, generate_reference, and field checkpoints flow through
field_out / field_in."""
import json
import math

import numpy as np
import pytest

from paper_2410_18944_b200 import harness

pytestmark = pytest.mark.gpu


def _cfg(tmp_path, **kw):
    d = {"preset": "neumann-strip-vlin", "grid": {"width": 32, "height": 32}, "wpp": 8,
         "sampler": "learnable_mis", "seed": 3}
    d.update(kw)
    return harness.parse_run_config(json.dumps(d))


def test_run_solve_outputs_and_log(gpu, tmp_path):
    ref_img = harness.generate_reference(_cfg(tmp_path), 0)  # analytic
    harness.write_csv(ref_img, str(tmp_path / "ref.csv"))
    cfg = _cfg(tmp_path, out=str(tmp_path / "u.csv"), out_pfm=str(tmp_path / "u.pfm"),
               out_png=str(tmp_path / "u.png"), log=str(tmp_path / "log.csv"),
               reference=str(tmp_path / "ref.csv"), field_out=str(tmp_path / "f.wgf"))
    res = harness.run_solve(cfg)
    assert np.all(res.image.cells["count"] == 8)  # escaped walks push 0 (wost.cpp:375-378)
    assert res.train_stats.steps >= 8 and res.train_stats.records_consumed > 0
    assert len(res.log) == 8 and all(math.isfinite(r.relmse) for r in res.log)
    assert res.log[-1].relmse == pytest.approx(harness.compute_relmse(res.image, ref_img), rel=1e-12)
    back = harness.read_csv(str(tmp_path / "u.csv"))
    assert np.array_equal(back.mean, res.image.mean)
    assert (tmp_path / "u.pfm").stat().st_size == 32 * 32 * 4 + len(b"Pf\n32 32\n-1.0\n")
    assert (tmp_path / "u.png").read_bytes()[:8] == b"\x89PNG\r\n\x1a\n"
    assert (tmp_path / "log.csv").read_text().splitlines()[0] == "wpp,relmse,seconds"
    # the checkpoint continues training where it stopped
    steps0 = res.field.state()[3]
    assert steps0 == res.train_stats.steps
    res2 = harness.run_solve(_cfg(tmp_path, wpp=2, field_in=str(tmp_path / "f.wgf")))
    assert res2.field.state()[3] == steps0 + res2.train_stats.steps


def test_ablation_and_equal_time(gpu, tmp_path):
    cfg = _cfg(tmp_path, wpp=16, grid={"width": 48, "height": 48})
    ref_img = harness.generate_reference(cfg, 0)
    rows = harness.run_ablation(cfg, ["uniform", "guiding_only", "fixed_mis", "learnable_mis"], ref_img)
    assert [r.mode for r in rows] == ["uniform", "guiding_only", "fixed_mis", "learnable_mis"]
    assert all(r.wpp == 16 and len(r.log) == 16 and math.isfinite(r.relmse) for r in rows)
    # relMSE falls with samples for every mode
    assert all(r.log[-1].relmse < r.log[0].relmse for r in rows)
    eq = harness.run_equal_time(cfg, ["uniform", "learnable_mis"], ref_img, seconds=0.2)
    by = {r.mode: r for r in eq}
    assert all(r.seconds >= 0.2 for r in eq)
    # a uniform step is far cheaper than a guided one: more samples in the same time
    assert by["uniform"].wpp > by["learnable_mis"].wpp >= 1
    with pytest.raises(ValueError):
        harness.run_ablation(cfg, [], ref_img)


def test_generate_reference_long_uniform_run(gpu, tmp_path):
    """Scene files have no analytic solution: generate_reference runs a long
    uniform solve on an independent seed (solver.cpp:169-190)."""
    from paper_2410_18944_b200 import scene_io
    from paper_2410_18944_b200.scene import make_preset
    path = tmp_path / "strip.json"
    path.write_text(scene_io.write_scene(make_preset("neumann-strip-vlin").scene))
    cfg = harness.parse_run_config(json.dumps({"scene": str(path), "grid": {"width": 16, "height": 16},
                                               "wpp": 4}))
    ref_img = harness.generate_reference(cfg, 512)
    assert np.all(ref_img.cells["count"] == 512)
    an = harness.generate_reference(_cfg(tmp_path, grid={"width": 16, "height": 16}), 0)
    short = harness.solve_points(harness.load_problem(cfg), cfg, ref_img.cell_centers(), 4).stats
    img4 = harness.make_image(16, 16, ref_img.bbox)
    img4.cells = short
    # uniform WoSt error ~ 1/wpp: 512 wpp is far closer to the analytic solution
    assert harness.compute_relmse(ref_img, an) < 0.25 * harness.compute_relmse(img4, an)
