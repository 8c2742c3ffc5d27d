"""Scene JSON files: load_scene / load_scene_file /
write_scene of proj/src/scene.cpp:99-368, onto the host Scene that
wostgpu_scene_create consumes (scene.py). Same keys, defaults, validation and
error messages (raised as SceneError, the reference's exception type).

The value table is ordered by name, like the reference's: nlohmann::json
objects iterate their keys sorted (std::map), so `values` is built in sorted
key order and a segment's value_index is the position of its name there.
Rasters are [height x width], row 0 at bbox.min.y ("data" row-major).
"""
from __future__ import annotations

import json
import math

import numpy as np

from . import abi
from ._lib import SceneError
from .scene import Scene, Value, default_epsilon_shell


def _fail(path, msg):
    raise SceneError(abi.WG_ERR_SCENE, f"scene: {path}: {msg}")


def _num(v):
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _vec2(j, path):
    if not isinstance(j, list) or len(j) != 2 or not _num(j[0]) or not _num(j[1]):
        _fail(path, "expected [x, y]")
    return float(j[0]), float(j[1])


def _bbox(j, path):
    if not isinstance(j, dict) or "min" not in j or "max" not in j:
        _fail(path, "expected {min:[x,y], max:[x,y]}")
    x0, y0 = _vec2(j["min"], path + ".min")
    x1, y1 = _vec2(j["max"], path + ".max")
    if not (x0 < x1) or not (y0 < y1):
        _fail(path, "min must be strictly below max")
    return (x0, y0, x1, y1)


def _raster(j, path):
    for k in ("width", "height", "bbox", "data"):
        if k not in j:
            _fail(path, "raster needs width, height, bbox, data")
    w, h = int(j["width"]), int(j["height"])
    bb = _bbox(j["bbox"], path + ".bbox")
    d = j["data"]
    if not isinstance(d, list) or not all(_num(v) for v in d):
        _fail(path + ".data", "expected a float array")
    if len(d) != w * h:  # RasterGrid size check (scene.cpp validate)
        _fail(path + ".data", f"expected {w * h} values, got {len(d)}")
    return np.asarray(d, dtype=np.float64).reshape(h, w), bb


def _value(j, path):
    if not isinstance(j, dict) or "type" not in j:
        _fail(path, "expected {type: ...}")
    t = j["type"]
    if t == "constant":
        if "value" not in j:
            _fail(path, "constant needs 'value'")
        return Value.constant(float(j["value"]))
    if t == "linear":
        return Value.linear(float(j.get("c0", 0.0)), float(j.get("cx", 0.0)), float(j.get("cy", 0.0)))
    if t == "raster":
        r, bb = _raster(j, path)
        return Value(abi.VALUE_RASTER, raster=r, raster_bbox=bb)
    _fail(path + ".type", f"unknown value type '{t}'")


def _source(j, path):
    if not isinstance(j, dict) or "type" not in j:
        _fail(path, "expected {type: ...}")
    t = j["type"]
    if t == "zero":
        return Value.zero()
    if t == "constant":
        if "value" not in j:
            _fail(path, "constant needs 'value'")
        return Value.constant(float(j["value"]))
    if t == "raster":
        r, bb = _raster(j, path)
        return Value(abi.VALUE_RASTER, raster=r, raster_bbox=bb)
    _fail(path + ".type", f"unknown source type '{t}'")


def load_scene(text: str) -> Scene:
    """load_scene (scene.cpp:226-290) + Scene::validate (scene.cpp:119-143)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneError(abi.WG_ERR_SCENE, f"scene: parse error at line {e.lineno}: {e.msg}") from None
    if not isinstance(doc, dict):
        _fail("$", "top level must be an object")
    if "bbox" not in doc:
        _fail("$", "missing 'bbox'")
    if "segments" not in doc:
        _fail("$", "missing 'segments'")
    bbox = _bbox(doc["bbox"], "bbox")
    eps = float(doc["epsilon_shell"]) if "epsilon_shell" in doc else default_epsilon_shell(bbox)
    names, values = [], []
    if "values" in doc:
        vals = doc["values"]
        if not isinstance(vals, dict):
            _fail("values", "expected an object")
        for name in sorted(vals):  # nlohmann::json object order
            names.append(name)
            values.append(_value(vals[name], "values." + name))
    source = _source(doc["source"], "source") if "source" in doc else Value.zero()
    segs = doc["segments"]
    if not isinstance(segs, list):
        _fail("segments", "expected an array")
    seg, kind, refs = [], [], []
    for i, js in enumerate(segs):
        path = f"segments[{i}]"
        if not isinstance(js, dict) or not all(k in js for k in ("a", "b", "kind", "value")):
            _fail(path, "segment needs a, b, kind, value")
        a = _vec2(js["a"], path + ".a")
        b = _vec2(js["b"], path + ".b")
        k = js["kind"]
        if k == "dirichlet":
            kind.append(abi.DIRICHLET)
        elif k == "neumann":
            kind.append(abi.NEUMANN)
        else:
            _fail(path + ".kind", "expected 'dirichlet' or 'neumann'")
        seg.append((a[0], a[1], b[0], b[1]))
        refs.append(str(js["value"]))
    # Scene::validate
    if not (eps > 0.0):
        raise SceneError(abi.WG_ERR_SCENE, f"epsilon_shell must be > 0 (got {eps:.6f})")
    if not seg:
        raise SceneError(abi.WG_ERR_SCENE, "scene has no boundary segments")
    for v, where in [(v, f"value '{n}'") for n, v in zip(names, values)] + [(source, "source")]:
        if v.type == abi.VALUE_RASTER and not np.all(np.isfinite(v.raster)):
            raise SceneError(abi.WG_ERR_SCENE, f"{where}: raster has non-finite entries")
    vidx = []
    for i, (s, r) in enumerate(zip(seg, refs)):
        where = f"segment {i}"
        if s[0] == s[2] and s[1] == s[3]:
            raise SceneError(abi.WG_ERR_SCENE, f"{where}: a == b (zero-length segment)")
        for x, y in ((s[0], s[1]), (s[2], s[3])):
            if not (bbox[0] <= x <= bbox[2] and bbox[1] <= y <= bbox[3]):
                raise SceneError(abi.WG_ERR_SCENE, f"{where}: endpoint outside scene bbox")
        if r not in names:
            raise SceneError(abi.WG_ERR_SCENE, f"{where}: value '{r}' is not defined")
        vidx.append(names.index(r))
    if abi.DIRICHLET not in kind:
        raise SceneError(abi.WG_ERR_SCENE, "scene has no Dirichlet segments: walks could never terminate")
    return Scene(bbox, eps, np.asarray(seg, dtype=np.float64), np.asarray(kind, dtype=np.int32),
                 np.asarray(vidx, dtype=np.int32), values, source, names)


def load_scene_file(path: str) -> Scene:
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise SceneError(abi.WG_ERR_SCENE, f"cannot open scene file '{path}'") from None
    return load_scene(text)


def _raster_json(r, bb):
    h, w = r.shape
    return {"width": w, "height": h, "bbox": {"min": [bb[0], bb[1]], "max": [bb[2], bb[3]]},
            "data": [float(v) for v in r.ravel()]}


def _value_json(v: Value):
    if v.type == abi.VALUE_CONSTANT:
        return {"type": "constant", "value": v.c0}
    if v.type == abi.VALUE_LINEAR:
        return {"type": "linear", "c0": v.c0, "cx": v.cx, "cy": v.cy}
    if v.type == abi.VALUE_RASTER:
        return dict(_raster_json(v.raster, v.raster_bbox), type="raster")
    raise SceneError(abi.WG_ERR_SCENE, "write_scene: analytic value spec is not serializable")


def write_scene(sc: Scene) -> str:
    """write_scene (scene.cpp:335-366)."""
    names = sc.value_names or [f"v{i}" for i in range(len(sc.values))]
    src = sc.source
    if src.type == abi.VALUE_ZERO:
        sj = {"type": "zero"}
    elif src.type == abi.VALUE_CONSTANT:
        sj = {"type": "constant", "value": src.c0}
    elif src.type == abi.VALUE_RASTER:
        sj = dict(_raster_json(src.raster, src.raster_bbox), type="raster")
    else:
        raise SceneError(abi.WG_ERR_SCENE, "write_scene: analytic source is not serializable")
    doc = {
        "bbox": {"min": [sc.bbox[0], sc.bbox[1]], "max": [sc.bbox[2], sc.bbox[3]]},
        "epsilon_shell": sc.epsilon_shell,
        "values": {n: _value_json(v) for n, v in zip(names, sc.values)},
        "source": sj,
        "segments": [{"a": [float(s[0]), float(s[1])], "b": [float(s[2]), float(s[3])],
                      "kind": "dirichlet" if k == abi.DIRICHLET else "neumann", "value": names[vi]}
                     for s, k, vi in zip(sc.seg, sc.kind, sc.value_index)],
    }
    return json.dumps(doc, indent=2)


def approx_equal_scenes(a: Scene, b: Scene) -> bool:
    """Same geometry, kinds, value bindings and epsilon (round-trip checks)."""
    return (a.bbox == b.bbox and math.isclose(a.epsilon_shell, b.epsilon_shell, rel_tol=0, abs_tol=0)
            and np.array_equal(a.seg, b.seg) and np.array_equal(a.kind, b.kind)
            and [a.values[i].eval(0.3, 0.7) for i in a.value_index if a.values[i].type != abi.VALUE_RASTER]
            == [b.values[i].eval(0.3, 0.7) for i in b.value_index if b.values[i].type != abi.VALUE_RASTER])
