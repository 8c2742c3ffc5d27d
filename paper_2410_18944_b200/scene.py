"""Host-side scene description and the built-in presets.

`Scene` mirrors wost::Scene (proj/include/wost/scene.hpp:70-96): boundary
segments with a kind and a value reference, a value table, a source field, a
bbox and the epsilon shell. The presets restate proj/src/presets.cpp; their
segment coordinates are built with the same double-precision expressions
(Python floats are IEEE doubles and math.cos/sin call the C library), so they
are bit-identical to the reference's (pinned in tests/test_scene.py).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import abi

K_PI = 3.14159265358979323846
K_TWO_PI = 2.0 * K_PI


@dataclass
class Value:
    """ValueSpec (scene.hpp:31-54): constant / linear / raster / analytic."""
    type: int = abi.VALUE_CONSTANT
    c0: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    analytic_id: int = 0
    raster: Optional[np.ndarray] = None  # [h, w] row 0 at bbox.min.y
    raster_bbox: tuple = (0.0, 0.0, 1.0, 1.0)

    @staticmethod
    def constant(v):
        return Value(abi.VALUE_CONSTANT, c0=float(v))

    @staticmethod
    def linear(c0, cx, cy):
        return Value(abi.VALUE_LINEAR, c0=float(c0), cx=float(cx), cy=float(cy))

    @staticmethod
    def analytic(fid):
        return Value(abi.VALUE_ANALYTIC, analytic_id=fid)

    @staticmethod
    def zero():
        return Value(abi.VALUE_ZERO)

    def to_c(self) -> abi.ValueSpec:
        v = abi.ValueSpec()
        v.type = self.type
        v.analytic_id = self.analytic_id
        v.c0, v.cx, v.cy = self.c0, self.cx, self.cy
        if self.type == abi.VALUE_RASTER:
            r = np.ascontiguousarray(self.raster, dtype=np.float64)
            self._keep = r
            v.raster_h, v.raster_w = r.shape
            v.raster_bbox = (C.c_double * 4)(*self.raster_bbox)
            v.raster_data = r.ctypes.data_as(C.POINTER(C.c_double))
        return v

    def eval(self, x, y):
        if self.type == abi.VALUE_CONSTANT:
            return self.c0
        if self.type == abi.VALUE_LINEAR:
            return self.c0 + self.cx * x + self.cy * y
        if self.type == abi.VALUE_ANALYTIC:
            if self.analytic_id == abi.ANALYTIC_X2_MINUS_Y2:
                return x * x - y * y
            return x * x + y * y - 1.0
        if self.type == abi.VALUE_RASTER:  # RasterGrid::at (scene.cpp:13-20): nearest cell, clamped
            g = np.asarray(self.raster, dtype=np.float64)
            h, w = g.shape
            b = self.raster_bbox
            u = (x - b[0]) / (b[2] - b[0])
            v = (y - b[1]) / (b[3] - b[1])
            i = min(max(int(u * w), 0), w - 1)
            j = min(max(int(v * h), 0), h - 1)
            return float(g[j, i])
        if self.type == abi.VALUE_ZERO:
            return 0.0
        raise NotImplementedError


@dataclass
class Scene:
    bbox: tuple
    epsilon_shell: float
    seg: np.ndarray  # [n, 4] ax ay bx by
    kind: np.ndarray  # [n] int32
    value_index: np.ndarray  # [n] int32
    values: List[Value]
    source: Value = field(default_factory=Value.zero)
    value_names: Optional[List[str]] = None  # Scene::values keys (scene JSON, scene_io.py)

    @property
    def n_segments(self):
        return int(self.seg.shape[0])

    def c_args(self):
        """Arguments of wostgpu_scene_create / {ref,orc}_scene_create."""
        self._vals = (abi.ValueSpec * max(1, len(self.values)))(*[v.to_c() for v in self.values])
        self._src = self.source.to_c()
        self._bbox = (C.c_double * 4)(*self.bbox)
        seg = np.ascontiguousarray(self.seg, dtype=np.float64)
        kind = np.ascontiguousarray(self.kind, dtype=np.int32)
        vi = np.ascontiguousarray(self.value_index, dtype=np.int32)
        self._arrs = (seg, kind, vi)
        return (abi.ptr(seg), abi.ptr(kind, C.c_int32), abi.ptr(vi, C.c_int32), C.c_int32(len(seg)),
                self._vals, C.c_int32(len(self.values)), C.byref(self._src), self._bbox,
                C.c_double(self.epsilon_shell))


def default_epsilon_shell(bbox):
    """scene.cpp:99-101"""
    return 1e-3 * math.sqrt((bbox[2] - bbox[0]) ** 2 + (bbox[3] - bbox[1]) ** 2)


class _Builder:
    def __init__(self, bbox, eps):
        self.bbox, self.eps = bbox, eps
        self.values, self.names = [], {}
        self.segs, self.kinds, self.vidx = [], [], []
        self.source = Value.zero()

    def value(self, name, v):
        self.names[name] = len(self.values)
        self.values.append(v)

    def polyline(self, pts, closed, kind, ref):  # add_polyline, presets.cpp:10-22
        n = len(pts)
        count = n if closed else n - 1
        for i in range(count):
            a, b = pts[i], pts[(i + 1) % n]
            self.segs.append((a[0], a[1], b[0], b[1]))
            self.kinds.append(kind)
            self.vidx.append(self.names[ref])

    def build(self):
        names = sorted(self.names, key=self.names.get)
        return Scene(self.bbox, self.eps, np.array(self.segs, dtype=np.float64),
                     np.array(self.kinds, dtype=np.int32), np.array(self.vidx, dtype=np.int32),
                     self.values, self.source, names)


def circle_points(center, radius, n):  # presets.cpp:24-31
    out = []
    for i in range(n):
        a = K_TWO_PI * i / n
        out.append((center[0] + radius * math.cos(a), center[1] + radius * math.sin(a)))
    return out


def _disk_scene(g: Value, source: Value, eps):  # presets.cpp:33-44
    b = _Builder((-1.1, -1.1, 1.1, 1.1), eps)
    b.value("g", g)
    b.source = source
    b.polyline(circle_points((0.0, 0.0), 1.0, 256), True, abi.DIRICHLET, "g")
    return b.build()


def _strip_scene(right: Value):  # presets.cpp:55-85
    bbox = (0.0, 0.0, 1.0, 1.0)
    b = _Builder(bbox, default_epsilon_shell(bbox))
    b.value("left", Value.constant(0.0))
    b.value("right", right)
    b.value("insulated", Value.constant(0.0))
    b.polyline([(0.0, 0.0), (0.0, 1.0)], False, abi.DIRICHLET, "left")
    b.polyline([(1.0, 0.0), (1.0, 1.0)], False, abi.DIRICHLET, "right")
    b.polyline([(0.0, 0.0), (1.0, 0.0)], False, abi.NEUMANN, "insulated")
    b.polyline([(0.0, 1.0), (1.0, 1.0)], False, abi.NEUMANN, "insulated")
    return b.build()


def _curves_scene():  # presets.cpp:99-165
    bbox = (0.0, 0.0, 1.0, 1.0)
    b = _Builder(bbox, default_epsilon_shell(bbox))
    b.value("white", Value.constant(1.0))
    b.value("black", Value.constant(0.0))
    b.value("insulated", Value.constant(0.0))
    b.polyline([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)], True, abi.NEUMANN, "insulated")
    b.polyline(circle_points((0.28, 0.64), 0.17, 64), True, abi.DIRICHLET, "white")
    b.polyline(circle_points((0.67, 0.40), 0.21, 64), True, abi.DIRICHLET, "black")
    b.polyline(circle_points((0.77, 0.79), 0.08, 48), True, abi.DIRICHLET, "white")
    b.polyline(circle_points((0.17, 0.25), 0.06, 48), True, abi.DIRICHLET, "black")
    spiral = []
    for i in range(97):
        t = i / 96
        a = 3.5 * K_PI * t
        r = 0.030 + 0.060 * t
        spiral.append((0.55 + r * math.cos(a), 0.84 + r * math.sin(a)))
    b.polyline(spiral, False, abi.DIRICHLET, "white")
    wave = []
    for i in range(65):
        t = i / 64
        wave.append((0.05 + 0.43 * t, 0.10 - 0.03 * t + 0.04 * math.sin(3.0 * K_PI * t)))
    b.polyline(wave, False, abi.DIRICHLET, "white")
    edge = []
    for i in range(65):
        t = i / 64
        edge.append((0.915 + 0.035 * math.sin(4.0 * K_PI * t), 0.55 + 0.40 * t))
    b.polyline(edge, False, abi.DIRICHLET, "black")
    zig = []
    for i in range(33):
        t = i / 32
        zig.append((0.05 + 0.25 * t, 0.93 + 0.025 * (1.0 if i % 2 else -1.0)))
    b.polyline(zig, False, abi.DIRICHLET, "white")
    bar = []
    for i in range(9):
        t = i / 8
        bar.append((0.55 + 0.20 * t, 0.08 + 0.06 * t))
    b.polyline(bar, False, abi.DIRICHLET, "black")
    return b.build()


def strip_vlin_solution(x, y):
    """Separable series of the neumann-strip-vlin problem, presets.cpp:169-184."""
    u = 0.5 * x
    n = 1
    while n < 2000:
        cn = -4.0 / (n * n * K_PI * K_PI)
        a = n * K_PI * x
        b = n * K_PI
        ratio = math.exp(a - b) * (1.0 - math.exp(-2.0 * a)) / (1.0 - math.exp(-2.0 * b))
        term = cn * ratio * math.cos(n * K_PI * y)
        u += term
        if abs(term) < 1e-14 and n > 64:
            break
        n += 2
    return u


@dataclass
class Preset:
    """wost::Preset (proj/include/wost/presets.hpp:14-20)."""
    name: str
    scene: Scene
    analytic: Optional[Callable[[float, float], float]]
    eval_bbox: tuple


def make_preset(name: str) -> Preset:
    """make_preset, presets.cpp:186-231."""
    if name == "harmonic-disk":
        sc = _disk_scene(Value.analytic(abi.ANALYTIC_X2_MINUS_Y2), Value.zero(), 1e-4)
        return Preset(name, sc, lambda x, y: x * x - y * y, (-0.55, -0.55, 0.55, 0.55))
    if name == "const-source-disk":
        sc = _disk_scene(Value.analytic(abi.ANALYTIC_R2_MINUS_1), Value.constant(4.0), 1e-6)
        return Preset(name, sc, lambda x, y: x * x + y * y - 1.0, (-0.55, -0.55, 0.55, 0.55))
    if name == "neumann-strip":
        sc = _strip_scene(Value.constant(1.0))
        return Preset(name, sc, lambda x, y: x, sc.bbox)
    if name == "neumann-strip-vlin":
        sc = _strip_scene(Value.linear(0.0, 0.0, 1.0))
        return Preset(name, sc, strip_vlin_solution, sc.bbox)
    if name == "curves":
        sc = _curves_scene()
        return Preset(name, sc, None, sc.bbox)
    raise ValueError(f"unknown preset '{name}'")


PRESET_NAMES = ["harmonic-disk", "const-source-disk", "neumann-strip", "neumann-strip-vlin", "curves"]


def cell_centers(width, height, bbox):
    """SolutionImage::cell_center, row-major j*width+i (proj/include/wost/image.hpp:26-31)."""
    ex, ey = bbox[2] - bbox[0], bbox[3] - bbox[1]
    i = np.arange(width, dtype=np.float64)
    j = np.arange(height, dtype=np.float64)
    xs = bbox[0] + (i + 0.5) / width * ex
    ys = bbox[1] + (j + 0.5) / height * ey
    out = np.empty((height, width, 2), dtype=np.float64)
    out[:, :, 0] = xs[None, :]
    out[:, :, 1] = ys[:, None]
    return out.reshape(-1, 2)


def analytic_image(preset: Preset, width, height, bbox=None):
    bbox = bbox or preset.eval_bbox
    pts = cell_centers(width, height, bbox)
    return np.array([preset.analytic(x, y) for x, y in pts], dtype=np.float64)


def relmse(est, ref):
    """compute_relmse, proj/src/image.cpp:211-230: mean (e-r)^2/(r^2+delta),
    delta = (0.01 max|ref|)^2."""
    est = np.asarray(est, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    max_abs = np.max(np.abs(ref))
    delta = 0.0001 * max_abs * max_abs
    d = est - ref
    denom = ref * ref + delta
    if np.any(denom <= 0.0):
        if np.any((denom <= 0.0) & (d != 0.0)):
            return math.inf
    ok = denom > 0.0
    return float(np.sum(d[ok] * d[ok] / denom[ok]) / est.size)
