"""Callers and formats of the path against the
reference's own implementation (oracle/_ref, ref_shim.cpp):

  * scene JSON: the reference's write_scene of each serialisable preset, read
    by our loader, gives the reference loader's segments / kinds / value
    bindings / bbox / epsilon exactly, and our preset geometry; invalid
    scenes raise SceneError with the reference's message;
  * result files: write_csv / write_pfm / write_png (+ tonemap sidecar) and
    the convergence log are byte-identical to the reference writers';
    compute_relmse agrees to the last bit;
  * run configs parse with the reference's keys, defaults and checks.
CPU only (no device calls)."""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2410_18944_b200 import abi, harness, scene_io
from paper_2410_18944_b200._lib import SceneError
from paper_2410_18944_b200.scene import make_preset


def _shim(ref):
    lib = ref.lib
    if not hasattr(lib, "ref_preset_scene_json"):
        pytest.skip("oracle/_ref built without the harness shim")
    lib.ref_preset_scene_json.restype = C.c_int64
    lib.ref_preset_scene_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
    lib.ref_load_scene_json.restype = C.c_int64
    lib.ref_load_scene_json.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
    lib.ref_write_image.restype = C.c_int
    lib.ref_write_image.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.c_void_p,
                                    C.c_char_p, C.c_char_p, C.c_char_p]
    lib.ref_compute_relmse.restype = C.c_double
    lib.ref_compute_relmse.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.ref_write_convergence_log.restype = C.c_int
    lib.ref_write_convergence_log.argtypes = [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                              C.POINTER(C.c_double), C.c_char_p]
    return lib


def _ref_scene_json(lib, name):
    n = lib.ref_preset_scene_json(name.encode(), None, 0)
    assert n > 0
    buf = C.create_string_buffer(n + 1)
    assert lib.ref_preset_scene_json(name.encode(), buf, n + 1) == n
    return buf.value.decode()


def _ref_load(ref, lib, text):
    cap = 4096
    seg = np.zeros((cap, 4))
    kind = np.zeros(cap, dtype=np.int32)
    vi = np.zeros(cap, dtype=np.int32)
    bbox = np.zeros(4)
    eps = np.zeros(1)
    n = lib.ref_load_scene_json(text.encode(), abi.ptr(seg), abi.ptr(kind, C.c_int32),
                                abi.ptr(vi, C.c_int32), cap, abi.ptr(bbox), abi.ptr(eps))
    if n < 0:
        return None, ref.fn("last_error")().decode()
    return (seg[:n], kind[:n], vi[:n], tuple(bbox), float(eps[0])), None


@pytest.mark.parametrize("name", ["neumann-strip", "neumann-strip-vlin", "curves"])
def test_scene_json_loader_matches_reference(ref, name):
    lib = _shim(ref)
    text = _ref_scene_json(lib, name)
    ours = scene_io.load_scene(text)
    (seg, kind, vi, bbox, eps), err = _ref_load(ref, lib, text)
    assert err is None
    assert np.array_equal(ours.seg, seg) and np.array_equal(ours.kind, kind)
    assert np.array_equal(ours.value_index, vi)
    assert ours.bbox == bbox and ours.epsilon_shell == eps
    # same geometry and boundary data as the preset it was written from
    p = make_preset(name).scene
    assert np.array_equal(ours.seg, p.seg) and np.array_equal(ours.kind, p.kind)
    for a, b in zip(ours.value_index, p.value_index):
        assert ours.values[a].eval(0.37, 0.61) == p.values[b].eval(0.37, 0.61)
    # and our writer round-trips
    again = scene_io.load_scene(scene_io.write_scene(ours))
    assert np.array_equal(again.seg, ours.seg) and np.array_equal(again.value_index, ours.value_index)


def _base_doc():
    return {"bbox": {"min": [0, 0], "max": [1, 1]},
            "values": {"g": {"type": "constant", "value": 1.0}, "h": {"type": "linear", "cy": 2.0}},
            "segments": [{"a": [0, 0], "b": [0, 1], "kind": "dirichlet", "value": "g"},
                         {"a": [0, 0], "b": [1, 0], "kind": "neumann", "value": "h"}]}


@pytest.mark.parametrize("mutate", [
    lambda d: d.pop("bbox"),
    lambda d: d.pop("segments"),
    lambda d: d["segments"][0].update(b=[0, 0]),
    lambda d: d["segments"][0].update(value="nope"),
    lambda d: d["segments"][0].update(a=[2, 0]),
    lambda d: d["segments"][0].update(kind="robin"),
    lambda d: d["segments"].pop(0),
    lambda d: d.update(bbox={"min": [1, 0], "max": [0, 1]}),
    lambda d: d["values"].update(g={"type": "cubic"}),
    lambda d: d.update(epsilon_shell=-1.0),
    lambda d: d.update(source={"type": "constant"}),
])
def test_scene_json_errors_match_reference(ref, mutate):
    lib = _shim(ref)
    doc = _base_doc()
    mutate(doc)
    text = json.dumps(doc)
    _, ref_err = _ref_load(ref, lib, text)
    assert ref_err is not None
    with pytest.raises(SceneError) as e:
        scene_io.load_scene(text)
    ours = str(e.value).split(": ", 1)[1]  # strip "wostgpu error N: "
    if "epsilon_shell" in ref_err:  # std::to_string formatting of the value
        assert ours.startswith("epsilon_shell must be > 0")
    else:
        assert ours == ref_err, (ours, ref_err)


def _image(rng, w=7, h=5):
    img = harness.make_image(w, h, (-0.25, 0.0, 1.5, 0.75))
    img.cells["mean"] = rng.normal(0.0, 2.0, w * h)
    img.cells["mean"][3] = 0.1  # a short decimal
    img.cells["count"] = rng.integers(0, 300, w * h)
    img.cells["m2"] = rng.uniform(0.0, 5.0, w * h)
    img.cells["escaped"] = rng.integers(0, 3, w * h)
    return img


def test_result_files_byte_identical_to_reference(ref, tmp_path):
    lib = _shim(ref)
    img = _image(np.random.default_rng(4))
    bb = np.array(img.bbox)
    paths = {k: (tmp_path / f"ref.{k}", tmp_path / f"ours.{k}") for k in ("csv", "pfm", "png")}
    assert lib.ref_write_image(img.width, img.height, abi.ptr(bb), C.c_void_p(img.cells.ctypes.data),
                               str(paths["csv"][0]).encode(), str(paths["pfm"][0]).encode(),
                               str(paths["png"][0]).encode()) == 0
    harness.write_csv(img, str(paths["csv"][1]))
    harness.write_pfm(img, str(paths["pfm"][1]))
    harness.write_png(img, str(paths["png"][1]))
    for k, (a, b) in paths.items():
        assert a.read_bytes() == b.read_bytes(), k
    sa = json.loads((tmp_path / "ref.png.json").read_text())
    sb = json.loads((tmp_path / "ours.png.json").read_text())
    assert sa == sb
    back = harness.read_csv(str(paths["csv"][1]))
    assert np.array_equal(back.mean, img.mean) and np.array_equal(back.cells["count"], img.cells["count"])
    assert np.allclose(back.variance_of_mean(), img.variance_of_mean(), rtol=1e-15, atol=0)
    assert np.array_equal(harness.read_pfm(str(paths["pfm"][1])).mean, img.mean.astype(np.float32))


def test_relmse_and_convergence_log_match_reference(ref, tmp_path):
    lib = _shim(ref)
    rng = np.random.default_rng(8)
    est, refv = rng.normal(0, 1, 35), rng.normal(0, 1, 35)
    a = harness.make_image(7, 5, (0, 0, 1, 1))
    b = harness.make_image(7, 5, (0, 0, 1, 1))
    a.cells["mean"], b.cells["mean"] = est, refv
    assert harness.compute_relmse(a, b) == lib.ref_compute_relmse(7, 5, abi.ptr(est), abi.ptr(refv))
    rows = [harness.LogRow(i + 1, float(rng.uniform(0, 0.1)), float(rng.uniform(0, 100))) for i in range(20)]
    rows[3].relmse = float("nan")
    harness.write_convergence_log(rows, str(tmp_path / "ours.log"))
    w = np.array([r.wpp for r in rows], dtype=np.int32)
    r = np.array([x.relmse for x in rows])
    s = np.array([x.seconds for x in rows])
    assert lib.ref_write_convergence_log(len(rows), abi.ptr(w, C.c_int32), abi.ptr(r), abi.ptr(s),
                                         str(tmp_path / "ref.log").encode()) == 0
    assert (tmp_path / "ours.log").read_bytes() == (tmp_path / "ref.log").read_bytes()


def test_run_config_parsing():
    cfg = harness.parse_run_config(json.dumps({
        "preset": "neumann-strip-vlin", "grid": {"width": 64, "height": 32,
                                                 "bbox": {"min": [0, 0], "max": [1, 0.5]}},
        "wpp": 17, "sampler": "fixed_mis", "fixed_c": 0.25, "train_until": 9, "seed": 5, "k": 4,
        "field": {"levels": [8, 16], "features": 2, "hidden": 32},
        "train": {"lr": 0.02, "minibatch": 1024, "max_records": 4096, "e_fraction": 0.1},
        "solver": {"rr_depth": 64, "reflect": False, "epsilon_shell": 1e-4, "r_min": 1e-5},
        "out": "a.csv", "log": "l.csv", "field_out": "f.wgf"}))
    assert (cfg.width, cfg.height, cfg.bbox, cfg.wpp, cfg.mode) == (64, 32, (0.0, 0.0, 1.0, 0.5), 17, "fixed_mis")
    assert (cfg.fixed_c, cfg.train_until, cfg.seed) == (0.25, 9, 5)
    assert list(cfg.field.level_res[:cfg.field.n_levels]) == [8, 16] and cfg.field.mixture_k == 4
    assert (cfg.field.features, cfg.field.hidden) == (2, 32)
    assert (cfg.train.lr, cfg.train.minibatch, cfg.train.max_records_per_round) == (0.02, 1024, 4096)
    sc = cfg.solver_config()
    assert (sc.rr_depth, sc.reflect_at_neumann, sc.mode, sc.fixed_c) == (64, 0, abi.MODE_FIXED_MIS, 0.25)
    assert (cfg.out_csv, cfg.log_path, cfg.field_out) == ("a.csv", "l.csv", "f.wgf")
    for bad in ({"wpp": 0}, {"fixed_c": 1.0}, {"sampler": "greedy"}, {"grid": {"width": 0}}):
        with pytest.raises(ValueError):
            harness.parse_run_config(json.dumps(dict({"preset": "curves"}, **bad)))
