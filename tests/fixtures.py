"""Test fixtures: a Python PCG32 identical to proj/include/wost/rng.hpp and the
reference unit tests' in-code scenes (proj/tests/test_geom2d.cpp:11-46,
proj/tests/test_wost.cpp:14-35), so the same random scenes and probes the
reference tests pin can be rebuilt here."""
import math

import numpy as np

from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.scene import Scene, Value, default_epsilon_shell

M64 = (1 << 64) - 1


def mix(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Rng:
    """PCG32, proj/include/wost/rng.hpp:9-78."""

    def __init__(self, seed=0x853C49E6748FEA9B, stream=0xDA3E39CB94B95BDB):
        self.state = 0
        self.inc = ((stream << 1) | 1) & M64
        self.next_u32()
        self.state = (self.state + seed) & M64
        self.next_u32()

    @staticmethod
    def for_walk(seed, point, wpp):
        a = mix(seed ^ mix(point))
        b = mix(a ^ mix((wpp + 0x632BE59BD9B4E019) & M64))
        return Rng(a, b)

    def next_u32(self):
        old = self.state
        self.state = (old * 6364136223846793005 + self.inc) & M64
        xs = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xs >> rot) | (xs << ((32 - rot) & 31))) & 0xFFFFFFFF

    def next_u64(self):
        hi = self.next_u32()
        return (hi << 32) | self.next_u32()

    def uniform(self, lo=None, hi=None):
        u = (self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_index(self, n):
        m = self.next_u32() * n
        lo = m & 0xFFFFFFFF
        if lo < n:
            t = ((1 << 32) - n) % n
            while lo < t:
                m = self.next_u32() * n
                lo = m & 0xFFFFFFFF
        return m >> 32


def segments_scene(segs, bbox, value=0.0):
    """segments_scene (test_geom2d.cpp:11-20): one constant value, no validate
    (epsilon_shell <= 0 selects that path in every implementation)."""
    seg = np.array([s[0] + s[1] for s in segs], dtype=np.float64).reshape(-1, 4)
    kind = np.array([s[2] for s in segs], dtype=np.int32)
    return Scene(tuple(bbox), 0.0, seg, kind, np.zeros(len(segs), dtype=np.int32),
                 [Value.constant(value)])


def random_scene(rng: Rng, n, mixed_kinds=True):
    """random_scene (test_geom2d.cpp:30-46)."""
    segs = []
    for _ in range(n):
        a = (rng.uniform(0, 1), rng.uniform(0, 1))
        d = (rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1))
        if d[0] == 0 and d[1] == 0:
            d = (0.01, 0.0)
        b = (min(max(a[0] + d[0], 0.0), 1.0), min(max(a[1] + d[1], 0.0), 1.0))
        if a == b:
            continue
        k = abi.NEUMANN if (mixed_kinds and rng.uniform() < 0.5) else abi.DIRICHLET
        segs.append((a, b, k))
    return segments_scene(segs, (0.0, 0.0, 1.0, 1.0))


def polygon_scene(center, radius, n, kind, value, bbox):
    """polygon_scene (test_wost.cpp:14-35), validated like the reference."""
    pts = []
    for i in range(n):
        a = 2.0 * 3.14159265358979323846 * i / n
        pts.append((center[0] + radius * math.cos(a), center[1] + radius * math.sin(a)))
    seg = np.array([pts[i] + pts[(i + 1) % n] for i in range(n)], dtype=np.float64)
    eps = 1e-3 * math.sqrt((bbox[2] - bbox[0]) ** 2 + (bbox[3] - bbox[1]) ** 2)
    return Scene(tuple(bbox), eps, seg, np.full(n, kind, dtype=np.int32),
                 np.zeros(n, dtype=np.int32), [Value.constant(value)])


def probes(rng: Rng, n, lo, hi):
    return np.array([(rng.uniform(lo, hi), rng.uniform(lo, hi)) for _ in range(n)])


# ---- scenes with Neumann flux and raster values (tests/test_gpu_values_train.py)
BOX = (0.0, 0.0, 1.0, 1.0)


def flux_scene():
    """Unit square: Dirichlet x = 0 (g = 0) and x = 1 (g = y); Neumann y = 0
    with constant flux h = 0.7 and y = 1 with linear flux h = 0.2 + 0.5 x."""
    seg = np.array([[0, 0, 1, 0], [1, 0, 1, 1], [1, 1, 0, 1], [0, 1, 0, 0]], dtype=np.float64)
    kind = np.array([abi.NEUMANN, abi.DIRICHLET, abi.NEUMANN, abi.DIRICHLET], dtype=np.int32)
    values = [Value.constant(0.7), Value.linear(0.0, 0.0, 1.0), Value.linear(0.2, 0.5, 0.0), Value.constant(0.0)]
    return Scene(BOX, default_epsilon_shell(BOX), seg, kind, np.array([0, 1, 2, 3], dtype=np.int32), values)


def raster_scene():
    """A 24-gon (radius 0.45) with raster Dirichlet values on half of its
    edges, a linear value on the rest, and a raster source term."""
    rng = np.random.default_rng(5)
    g = Value(abi.VALUE_RASTER, raster=rng.uniform(-1.0, 2.0, (5, 7)), raster_bbox=(0.0, 0.0, 1.0, 1.0))
    f = Value(abi.VALUE_RASTER, raster=rng.uniform(0.0, 3.0, (6, 6)), raster_bbox=(0.0, 0.0, 1.0, 1.0))
    n = 24
    ang = 2.0 * np.pi * np.arange(n) / n
    pts = np.stack([0.5 + 0.45 * np.cos(ang), 0.5 + 0.45 * np.sin(ang)], 1)
    seg = np.concatenate([pts, np.roll(pts, -1, 0)], 1)
    kind = np.full(n, abi.DIRICHLET, dtype=np.int32)
    vi = np.array([0 if i % 2 == 0 else 1 for i in range(n)], dtype=np.int32)
    return Scene(BOX, default_epsilon_shell(BOX), seg, kind, vi, [g, Value.linear(0.5, 1.0, -1.0)], source=f)


