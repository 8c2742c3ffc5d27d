"""3D test scenes and probes (no reference counterpart; SURVEY.md §8 a′).

* soup_scene: random small triangles inside the unit box, random kinds —
  stresses the BVHs and the silhouette-edge index (every Neumann edge of a
  soup is an open boundary edge).
* jittered_box: the box-strip-vlin mesh with every interior face vertex
  moved by a random offset (the same offset wherever the vertex is shared),
  so shared Neumann edges are creases and the facing test decides.
* numpy brute force for closest point / first hit, used to check the oracle's
  BVH traversal.
"""
import numpy as np

from paper_2410_18944_b200 import abi
from paper_2410_18944_b200.scene3 import VALUE_CONSTANT, VALUE_LINEAR, Scene3, make_preset3


def soup_scene(seed, n, size=0.08):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.1, 0.9, (n, 1, 3))
    tris = c + rng.uniform(-size, size, (n, 3, 3))
    kind = rng.integers(0, 2, n).astype(np.int32)
    values = [(VALUE_CONSTANT, 0.0, 0.0, 0.0, 0.0), (VALUE_LINEAR, 0.5, 1.0, -2.0, 0.25)]
    vidx = np.where(kind == abi.DIRICHLET, 1, 0).astype(np.int32)
    return Scene3(tris.astype(np.float64), kind, vidx, values, (0.0, 0.0, 0.0, 1.0, 1.0, 1.0), 1e-3)


def jittered_box(seed, n=8, amp=0.02):
    sc = make_preset3("box-strip-vlin", n=n).scene
    rng = np.random.default_rng(seed)
    flat = sc.tris.reshape(-1, 3).copy()
    moved = {}
    for i, p in enumerate(flat):
        k = tuple(p)
        if k not in moved:
            on = [v == 0.0 or v == 1.0 for v in p]
            d = np.zeros(3)
            if sum(on) == 1:  # interior to one face: slide in-plane, push inwards
                ax = on.index(True)
                d = rng.uniform(-amp, amp, 3)
                d[ax] = (1.0 if p[ax] == 0.0 else -1.0) * rng.uniform(0.0, amp)
            moved[k] = d
        flat[i] = p + moved[k]
    return Scene3(flat.reshape(-1, 3, 3), sc.kind.copy(), sc.value_index.copy(), list(sc.values), sc.bbox,
                  sc.eps)


def probes3(seed, n, lo=0.02, hi=0.98):
    return np.random.default_rng(seed).uniform(lo, hi, (n, 3))


def directions3(seed, n):
    d = np.random.default_rng(seed).normal(size=(n, 3))
    return d / np.linalg.norm(d, axis=1)[:, None]


def brute_closest(tris, x):
    """Exact-enough distance from each probe to each triangle (fp64 numpy):
    min over the in-plane projection (when inside) and the three edges."""
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    out = np.empty((len(x), len(tris)))
    n = np.cross(b - a, c - a)
    nn = n / np.linalg.norm(n, axis=1)[:, None]

    def seg_d2(p, s0, s1):
        ab = s1 - s0
        t = np.clip(np.einsum("ij,ij->i", p - s0, ab) / np.einsum("ij,ij->i", ab, ab), 0.0, 1.0)
        q = s0 + t[:, None] * ab
        return np.sum((p - q) ** 2, axis=1)

    for i, p in enumerate(x):
        P = np.broadcast_to(p, a.shape)
        h = np.einsum("ij,ij->i", P - a, nn)
        q = P - h[:, None] * nn
        # barycentric inside test
        v0, v1, v2 = c - a, b - a, q - a
        d00 = np.einsum("ij,ij->i", v0, v0)
        d01 = np.einsum("ij,ij->i", v0, v1)
        d11 = np.einsum("ij,ij->i", v1, v1)
        d20 = np.einsum("ij,ij->i", v2, v0)
        d21 = np.einsum("ij,ij->i", v2, v1)
        den = d00 * d11 - d01 * d01
        u = (d11 * d20 - d01 * d21) / den
        v = (d00 * d21 - d01 * d20) / den
        inside = (u >= 0) & (v >= 0) & (u + v <= 1)
        d2 = np.minimum(np.minimum(seg_d2(P, a, b), seg_d2(P, b, c)), seg_d2(P, c, a))
        d2 = np.where(inside, h * h, d2)
        out[i] = d2
    return out


def brute_ray(tris, o, d, t_eps, t_max):
    """First hit t per ray (inf on a miss) by Moller-Trumbore over all triangles."""
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    e1, e2 = b - a, c - a
    ts = np.full(len(o), np.inf)
    for i in range(len(o)):
        p = np.cross(d[i], e2)
        det = np.einsum("ij,ij->i", e1, p)
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = 1.0 / det
            s = o[i] - a
            u = np.einsum("ij,ij->i", s, p) * inv
            q = np.cross(s, e1)
            v = (q @ d[i]) * inv
            t = np.einsum("ij,ij->i", e2, q) * inv
        ok = (det != 0) & (u >= 0) & (u <= 1) & (v >= 0) & (u + v <= 1) & (t > t_eps) & (t <= t_max)
        if ok.any():
            ts[i] = t[ok].min()
    return ts
