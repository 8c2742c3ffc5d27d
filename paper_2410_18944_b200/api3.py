"""Python surface of the 3D path (include/wostgpu3.h; SURVEY.md §8 a′): the
3D analogues of api.Accel / GuidingField / Solver over triangle-mesh scenes
(scene3.Scene3). Everything runs on the GPU through libwostgpu.so; there is
no CPU fallback."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from ._lib import check, load

MLP_EXACT, MLP_TENSOR = 0, 1
D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)


def _d(a):
    return a.ctypes.data_as(D)


def _i(a):
    return a.ctypes.data_as(I32)


def _xyz(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != 3:
        raise ValueError("points must be [n, 3]")
    return x


def mixture3f_pdf(raw, nu):
    """The tensor-core 3D direction kernel's fp32 mixture math (diagnostic):
    decode each raw row (41 floats, K = 8) and evaluate the d = 3 mixture pdf
    at the unit direction nu[i]; returns (pdf [n], c [n])."""
    raw = np.ascontiguousarray(raw, dtype=np.float32)
    nu = _xyz(nu)
    if raw.ndim != 2 or raw.shape[1] != 41 or len(raw) != len(nu):
        raise ValueError("raw must be [n, 41] with one direction per row")
    out = np.zeros((raw.shape[0], 2))
    check(load().wostgpu_mixture3f_pdf(raw.shape[0], raw.ctypes.data_as(C.POINTER(C.c_float)), _d(nu), _d(out)))
    return out[:, 0], out[:, 1]


class Accel3:
    """Triangle-mesh scene with its per-kind BVHs and silhouette-edge index on
    one GPU (the 3D analogue of Accel, proj/src/geom2d.cpp:80-140)."""

    def __init__(self, scene):
        self.scene = scene
        h = C.c_void_p()
        check(load().wostgpu_scene3_create(*scene.c_args(), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            load().wostgpu_scene3_destroy(self.h)
            self.h = None

    def info(self):
        t = C.c_double()
        nodes = (C.c_int64 * 3)()
        a, c = C.c_int64(), C.c_int64()
        check(load().wostgpu_scene3_info(self.h, C.byref(t), nodes, C.byref(a), C.byref(c)))
        return {"t_epsilon": t.value, "nodes": list(nodes), "sil_always": a.value, "sil_crease": c.value}

    def closest_point(self, x, kinds=abi.KIND_ALL):
        x = _xyz(x)
        n = len(x)
        pt, d, tri = np.zeros((n, 3)), np.zeros(n), np.zeros(n, dtype=np.int32)
        check(load().wostgpu_closest_point3(self.h, n, _d(x), kinds, _d(pt), _d(d), _i(tri)))
        return pt, d, tri

    def closest_silhouette(self, x):
        x = _xyz(x)
        d = np.zeros(len(x))
        check(load().wostgpu_closest_silhouette3(self.h, len(x), _d(x), _d(d)))
        return d

    def ray_first_hit(self, origin, direction, t_max, kinds=abi.KIND_ALL, exclude=None):
        o, dr = _xyz(origin), _xyz(direction)
        n = len(o)
        tm = np.ascontiguousarray(np.broadcast_to(t_max, (n,)), dtype=np.float64)
        ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.int32)
        t, pt, nrm = np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3))
        tri, kind = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        check(load().wostgpu_ray_first_hit3(self.h, n, _d(o), _d(dr), _d(tm), kinds,
                                            None if ex is None else _i(ex), _d(t), _d(pt), _d(nrm),
                                            _i(tri), _i(kind)))
        return t, pt, nrm, tri, kind

    def star_radius(self, x, r_min):
        x = _xyz(x)
        r = np.zeros(len(x))
        check(load().wostgpu_star_radius3(self.h, len(x), _d(x), r_min, _d(r)))
        return r


class GuidingField3:
    """3D guiding field: dense res^3 x F grids + the MLP, output 5K + 1."""

    def __init__(self, cfg: abi.FieldConfig, bbox, seed):
        self.cfg = cfg
        self.bbox = tuple(float(v) for v in bbox)
        h = C.c_void_p()
        check(load().wostgpu_field3_create(C.byref(cfg), (C.c_double * 6)(*self.bbox), seed, C.byref(h)))
        self.h = h
        n = C.c_int64()
        check(load().wostgpu_field_param_count(self.h, C.byref(n)))
        self.n_params = n.value

    def __del__(self):
        if getattr(self, "h", None):
            load().wostgpu_field_destroy(self.h)
            self.h = None

    @property
    def output_dim(self):
        return 5 * self.cfg.mixture_k + 1

    def params(self):
        p = np.zeros(self.n_params, dtype=np.float32)
        check(load().wostgpu_field_get_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)), None, None, None))
        return p

    def state(self):
        p = np.zeros(self.n_params, dtype=np.float32)
        m, v = np.zeros(self.n_params), np.zeros(self.n_params)
        st = C.c_int64()
        check(load().wostgpu_field_get_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)), _d(m), _d(v),
                                             C.byref(st)))
        return p, m, v, st.value

    def set_params(self, p):
        _, m, v, st = self.state()
        self.set_state(p, m, v, st)

    def set_state(self, p, m, v, steps):
        p = np.ascontiguousarray(p, dtype=np.float32)
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        check(load().wostgpu_field_set_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)), _d(m), _d(v), steps))

    def save(self, path):
        """Checkpoint in the WGF1 layout (GuidingField::save,
        proj/src/guide_field.cpp:351-372) with magic "WGF3" and a 3D bbox
        (6 doubles): WGF1 itself is 2D-only."""
        p, m, v, steps = self.state()
        c = self.cfg
        with open(path, "wb") as f:
            f.write(b"WGF3")
            hdr = [1, c.n_levels] + [c.level_res[i] for i in range(c.n_levels)]
            hdr += [c.features, c.hidden, c.mixture_k, c.mixture_dim]
            f.write(np.array(hdr, dtype="<u4").tobytes())
            f.write(np.array(self.bbox, dtype="<f8").tobytes())
            f.write(np.array([steps], dtype="<i8").tobytes())
            f.write(np.array([len(p)], dtype="<u8").tobytes())
            f.write(p.astype("<f4").tobytes())
            f.write(m.astype("<f8").tobytes())
            f.write(v.astype("<f8").tobytes())

    @classmethod
    def load(cls, path):
        with open(path, "rb") as f:
            data = f.read()
        if data[:4] != b"WGF3":
            raise ValueError("3D guiding field checkpoint: bad magic")
        off = 4
        ver, nl = (int(x) for x in np.frombuffer(data, "<u4", 2, off))
        if ver != 1:
            raise ValueError("3D guiding field checkpoint: unknown version")
        off += 8
        res = [int(r) for r in np.frombuffer(data, "<u4", nl, off)]
        off += 4 * nl
        feat, hid, k, dim = (int(x) for x in np.frombuffer(data, "<u4", 4, off))
        off += 16
        bbox = tuple(float(x) for x in np.frombuffer(data, "<f8", 6, off))
        off += 48
        steps = int(np.frombuffer(data, "<i8", 1, off)[0])
        off += 8
        n = int(np.frombuffer(data, "<u8", 1, off)[0])
        off += 8
        field = cls(abi.field_config(tuple(res), features=feat, hidden=hid, mixture_k=k, mixture_dim=dim), bbox, 0)
        if n != field.n_params or len(data) < off + 20 * n:
            raise ValueError("3D guiding field checkpoint: size mismatch or truncated")
        p = np.frombuffer(data, "<f4", n, off)
        m = np.frombuffer(data, "<f8", n, off + 4 * n)
        v = np.frombuffer(data, "<f8", n, off + 12 * n)
        field.set_state(p, m, v, steps)
        return field

    def eval_batch(self, x, mlp=MLP_EXACT):
        x = _xyz(x)
        out = np.zeros((len(x), self.output_dim))
        check(load().wostgpu_field3_eval_batch(self.h, len(x), _d(x), _d(out), mlp))
        return out


class Solver3:
    """solve_batch / Engine over 3D evaluation points (wostgpu_solver3_*)."""

    def __init__(self, accel: Accel3, field: GuidingField3 | None, cfg: abi.SolverConfig, mlp=None):
        self.accel, self.field, self.cfg = accel, field, cfg
        h = C.c_void_p()
        check(load().wostgpu_solver3_create(accel.h, field.h if field else None, C.byref(cfg), C.byref(h)))
        self.h = h
        self.n_points = 0
        if mlp is not None:
            self.set_mlp(mlp)

    def set_mlp(self, mlp):
        check(load().wostgpu_solver3_set_mlp(self.h, mlp))

    def __del__(self):
        if getattr(self, "h", None):
            load().wostgpu_solver3_destroy(self.h)
            self.h = None

    def set_points(self, x, global_offset=0):
        x = _xyz(x)
        self.n_points = len(x)
        check(load().wostgpu_solver3_set_points(self.h, len(x), _d(x), global_offset))

    def stats(self):
        st = np.zeros(self.n_points, dtype=abi.POINT_STATS_DTYPE)
        check(load().wostgpu_solver3_get_stats(self.h, C.c_void_p(st.ctypes.data)))
        return st

    def solve_rounds(self, seed, wpp_first, n_rounds, collect=False):
        check(load().wostgpu_solver3_solve_rounds(self.h, seed, wpp_first, n_rounds, int(collect)))

    def walks(self):
        n = self.n_points
        est, esc, steps = np.zeros(n), np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        check(load().wostgpu_solver3_fetch_walks(self.h, _d(est), _i(esc), _i(steps)))
        return est, esc, steps

    def records(self):
        n = C.c_int64()
        check(load().wostgpu_solver3_fetch_records(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=abi.GUIDE_RECORD3_DTYPE)
        check(load().wostgpu_solver3_fetch_records(self.h, C.c_void_p(out.ctypes.data), n.value, C.byref(n)))
        return out[: n.value]

    def counters(self):
        v = [C.c_int64() for _ in range(4)]
        check(load().wostgpu_solver3_counters(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("walks", "steps", "escaped", "records"), (x.value for x in v)))

    def train_round(self, cfg: abi.TrainConfig, rnd):
        st = abi.TrainStats()
        check(load().wostgpu_solver3_train_round(self.h, C.byref(cfg), rnd, C.byref(st)))
        return st

    def field_grad(self, records, cfg: abi.TrainConfig):
        recs = np.ascontiguousarray(records, dtype=abi.GUIDE_RECORD3_DTYPE)
        g = np.zeros(self.field.n_params)
        check(load().wostgpu_solver3_field_grad(self.h, C.c_void_p(recs.ctypes.data), len(recs), C.byref(cfg),
                                                _d(g)))
        return g

    def run(self, seed, wpp, train_until=256, train_cfg: abi.TrainConfig | None = None):
        st = abi.TrainStats()
        ms = C.c_double()
        check(load().wostgpu_solver3_run(self.h, seed, wpp, train_until,
                                         C.byref(train_cfg) if train_cfg is not None else None,
                                         C.byref(st), C.byref(ms)))
        return st, ms.value

    def run_profile(self):
        w, t = C.c_double(), C.c_double()
        v = [C.c_int64() for _ in range(4)]
        check(load().wostgpu_solver3_run_profile(self.h, C.byref(w), C.byref(t), *[C.byref(x) for x in v]))
        out = dict(zip(("walks", "steps", "escaped", "train_steps"), (x.value for x in v)))
        out["walk_ms"], out["train_ms"] = w.value, t.value
        return out

    def reserve_records(self, n):
        """Record arena of at least n records per collecting round (a round
        that overflows the arena fails its call instead of training on a
        short-walk-biased subset)."""
        check(load().wostgpu_solver3_reserve_records(self.h, int(n)))

    def attach_comm(self, unique_id: bytes, nranks, rank):
        check(load().wostgpu_solver3_attach_comm(self.h, unique_id, nranks, rank))
