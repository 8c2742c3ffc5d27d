"""3D triangle-mesh scenes for configs 4-5 (SURVEY.md §8 a′, §8 d).

The reference has no 3D scene, so the presets here are builder-defined
(SURVEY.md §8 d, cfg 4): the unit box [0,1]^3 with every face split into
n x n squares of two triangles (6 * 2 * n^2 triangles; n = 91 gives 99,372),
Dirichlet on x = 0 (g = 0) and x = 1 (g = y), insulated (Neumann, h = 0) on
the four lateral faces. The solution is z-independent and equals the 2D
neumann-strip-vlin series (proj/src/presets.cpp:169-184), so relMSE against
an analytic solution is available on any slice. Faces are wound so that
normals point out of the domain; shared vertices are bit-identical (every
coordinate is i / n from one formula), which the silhouette-edge index keys
on.

`box-strip-vlin-obstacle` adds an insulated box [0.35,0.65] x [0.35,0.65] x
[0.3,0.7] inside the domain (normals pointing into the obstacle): its 12
edges are crease silhouettes. No analytic solution; it is the GPU-vs-oracle
parity scene for the silhouette and reflection paths.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import abi
from .scene import strip_vlin_solution

VALUE_CONSTANT, VALUE_LINEAR = 0, 1


@dataclass
class Scene3:
    tris: np.ndarray        # [n, 3, 3] float64 vertices a, b, c
    kind: np.ndarray        # [n] int32 (abi.DIRICHLET / abi.NEUMANN)
    value_index: np.ndarray  # [n] int32 into values
    values: list = field(default_factory=list)  # (type, c0, cx, cy, cz)
    bbox: tuple = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    eps: float = 1e-3
    source: Optional[tuple] = None  # (type, c0, cx, cy, cz) of f; None: no source

    @property
    def n_tris(self):
        return int(self.tris.shape[0])

    def c_values(self):
        arr = (abi.Value3Spec * max(len(self.values), 1))()
        for i, (t, c0, cx, cy, cz) in enumerate(self.values):
            arr[i] = abi.Value3Spec(t, 0, c0, cx, cy, cz)
        return arr

    def c_args(self):
        """(tri, kind, value_index, n, values, n_values, source, bbox, eps) as
        ctypes arguments (arrays kept alive on the scene object)."""
        tri = np.ascontiguousarray(self.tris.reshape(-1), dtype=np.float64)
        kind = np.ascontiguousarray(self.kind, dtype=np.int32)
        vi = np.ascontiguousarray(self.value_index, dtype=np.int32)
        bbox = np.ascontiguousarray(self.bbox, dtype=np.float64)
        vals = self.c_values()
        src = None
        if self.source is not None:
            t, c0, cx, cy, cz = self.source
            src = abi.Value3Spec(t, 0, c0, cx, cy, cz)
        self._keep = (tri, kind, vi, bbox, vals, src)
        return (abi.ptr(tri), abi.ptr(kind, C.c_int32), abi.ptr(vi, C.c_int32), self.n_tris, vals,
                len(self.values), C.byref(src) if src is not None else None, abi.ptr(bbox), self.eps)


def box_mesh(n, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), outward=True):
    """Faces of an axis-aligned box as [(axis, side, tris)], 2 n^2 tris each."""
    faces = []
    for axis in range(3):
        for side in (lo[axis], hi[axis]):
            # per-axis extents: faces are squares of the box's own extents
            u, v = (axis + 1) % 3, (axis + 2) % 3
            tr = []
            tu = lo[u] + (hi[u] - lo[u]) * (np.arange(n + 1, dtype=np.float64) / n)
            tv = lo[v] + (hi[v] - lo[v]) * (np.arange(n + 1, dtype=np.float64) / n)
            plus = (side == hi[axis]) == outward
            for i in range(n):
                for j in range(n):
                    def P(a, b):
                        p = [0.0, 0.0, 0.0]
                        p[axis] = side
                        p[u] = tu[a]
                        p[v] = tv[b]
                        return p
                    p00, p10, p11, p01 = P(i, j), P(i + 1, j), P(i + 1, j + 1), P(i, j + 1)
                    if plus:
                        tr += [(p00, p10, p11), (p00, p11, p01)]
                    else:
                        tr += [(p00, p11, p10), (p00, p01, p11)]
            faces.append((axis, side, tr))
    return faces


def _box_strip_scene(n, obstacle=False, obstacle_n=4):
    values = [(VALUE_CONSTANT, 0.0, 0.0, 0.0, 0.0), (VALUE_LINEAR, 0.0, 0.0, 1.0, 0.0)]
    tris, kind, vidx = [], [], []
    for axis, side, tr in box_mesh(n):
        if axis == 0:  # x faces: Dirichlet g = 0 (x = 0), g = y (x = 1)
            k, v = abi.DIRICHLET, (0 if side == 0.0 else 1)
        else:
            k, v = abi.NEUMANN, 0
        tris += tr
        kind += [k] * len(tr)
        vidx += [v] * len(tr)
    if obstacle:
        for _, _, tr in box_mesh(obstacle_n, (0.35, 0.35, 0.3), (0.65, 0.65, 0.7), outward=False):
            tris += tr
            kind += [abi.NEUMANN] * len(tr)
            vidx += [0] * len(tr)
    return Scene3(np.asarray(tris, dtype=np.float64), np.asarray(kind, dtype=np.int32),
                  np.asarray(vidx, dtype=np.int32), values, (0.0, 0.0, 0.0, 1.0, 1.0, 1.0),
                  1e-3 * math.sqrt(3.0))


def _box_poisson_scene(n):
    """u = x^2: Delta u = 2 = f (the reference's sign, const-source-disk), g = 0
    at x = 0 and 1 at x = 1, insulated lateral faces (du/dn = 0 there)."""
    sc = _box_strip_scene(n)
    sc.values = [(VALUE_CONSTANT, 0.0, 0.0, 0.0, 0.0), (VALUE_CONSTANT, 1.0, 0.0, 0.0, 0.0)]
    sc.source = (VALUE_CONSTANT, 2.0, 0.0, 0.0, 0.0)
    return sc


def _box_flux_scene(n):
    """u = y: Dirichlet g = y on the x faces, Neumann flux h = du/dn (outward
    normal) = -1 on y = 0, +1 on y = 1, 0 on the z faces."""
    values = [(VALUE_CONSTANT, 0.0, 0.0, 0.0, 0.0), (VALUE_LINEAR, 0.0, 0.0, 1.0, 0.0),
              (VALUE_CONSTANT, -1.0, 0.0, 0.0, 0.0), (VALUE_CONSTANT, 1.0, 0.0, 0.0, 0.0)]
    tris, kind, vidx = [], [], []
    for axis, side, tr in box_mesh(n):
        if axis == 0:
            k, v = abi.DIRICHLET, 1
        elif axis == 1:
            k, v = abi.NEUMANN, (2 if side == 0.0 else 3)
        else:
            k, v = abi.NEUMANN, 0
        tris += tr
        kind += [k] * len(tr)
        vidx += [v] * len(tr)
    return Scene3(np.asarray(tris, dtype=np.float64), np.asarray(kind, dtype=np.int32),
                  np.asarray(vidx, dtype=np.int32), values, (0.0, 0.0, 0.0, 1.0, 1.0, 1.0), 1e-3 * math.sqrt(3.0))


@dataclass
class Preset3:
    name: str
    scene: Scene3
    analytic: Optional[Callable[[float, float, float], float]]
    slice_bbox: tuple  # (x0, y0, x1, y1) of the evaluation slice
    slice_z: float


def make_preset3(name: str, n: int = 91) -> Preset3:
    """cfg 4 domain (SURVEY.md §8 d): n = 91 -> 99,372 triangles."""
    if name == "box-strip-vlin":
        sc = _box_strip_scene(n)
        return Preset3(name, sc, lambda x, y, z: strip_vlin_solution(x, y), (0.0, 0.0, 1.0, 1.0), 0.5)
    if name == "box-strip-vlin-obstacle":
        sc = _box_strip_scene(n, obstacle=True)
        return Preset3(name, sc, None, (0.0, 0.0, 1.0, 1.0), 0.5)
    if name == "box-poisson":
        return Preset3(name, _box_poisson_scene(n), lambda x, y, z: x * x, (0.0, 0.0, 1.0, 1.0), 0.5)
    if name == "box-flux":
        return Preset3(name, _box_flux_scene(n), lambda x, y, z: y, (0.0, 0.0, 1.0, 1.0), 0.5)
    raise ValueError(f"unknown 3D preset '{name}'")


PRESET3_NAMES = ["box-strip-vlin", "box-strip-vlin-obstacle", "box-poisson", "box-flux"]


def slice_points(width, height, bbox=(0.0, 0.0, 1.0, 1.0), z=0.5):
    """Cell centres of a width x height slice at height z, row-major j*width+i."""
    ex, ey = bbox[2] - bbox[0], bbox[3] - bbox[1]
    xs = bbox[0] + (np.arange(width, dtype=np.float64) + 0.5) / width * ex
    ys = bbox[1] + (np.arange(height, dtype=np.float64) + 0.5) / height * ey
    out = np.empty((height, width, 3), dtype=np.float64)
    out[:, :, 0] = xs[None, :]
    out[:, :, 1] = ys[:, None]
    out[:, :, 2] = z
    return out.reshape(-1, 3)


def strip_vlin_np(x, y):
    """Vectorised strip_vlin_solution (presets.cpp:169-184): the same series
    summed over every odd n < 2000 whose largest term is still above 1e-14
    (the per-point early exit only drops terms below that)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    u = 0.5 * x
    for n in range(1, 2000, 2):
        cn = -4.0 / (n * n * math.pi * math.pi)
        a = n * math.pi * x
        b = n * math.pi
        ratio = np.exp(a - b) * (1.0 - np.exp(-2.0 * a)) / (1.0 - math.exp(-2.0 * b))
        term = cn * ratio * np.cos(n * math.pi * y)
        u = u + term
        if n > 64 and np.max(np.abs(term)) < 1e-14:
            break
    return u


def analytic_slice(preset: Preset3, width, height):
    pts = slice_points(width, height, preset.slice_bbox, preset.slice_z)
    return strip_vlin_np(pts[:, 0], pts[:, 1])
