"""Python mirror of the reference's wost:: API for the guided WoSt hot path,
running on the B200 through the C-ABI (include/wostgpu.h).

Names, argument meaning and error behaviour follow the reference headers:
  Accel          proj/include/wost/geom2d.hpp:38-91
  GuidingField   proj/include/wost/guide_field.hpp:37-96
  solve_batch    proj/include/wost/wost.hpp:160-163
  train_batch    proj/include/wost/guide_train.hpp:104-105
  Engine/run     proj/src/solver.cpp:53-167 (see harness.py)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from ._lib import check, init, load
from .scene import Scene

MLP_EXACT, MLP_TENSOR = 0, 1


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _xy(xy):
    return np.ascontiguousarray(np.asarray(xy, dtype=np.float64).reshape(-1, 2))


class Accel:
    """wost::Accel over a Scene: the device scene + BVH (geom2d.hpp:38)."""

    def __init__(self, scene: Scene, device=None):
        init(device)
        self.scene = scene
        h = C.c_void_p()
        check(load().wostgpu_scene_create(*scene.c_args(), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            load().wostgpu_scene_destroy(self.h)
            self.h = None

    def _info(self):
        t = C.c_double()
        f = C.c_int32()
        box = (C.c_double * 4)()
        check(load().wostgpu_scene_info(self.h, C.byref(t), C.byref(f), box))
        return t.value, bool(f.value), tuple(box)

    @property
    def t_epsilon(self):
        return self._info()[0]

    @property
    def root_box(self):
        return self._info()[2]

    @property
    def has_neumann_flux(self):
        return self._info()[1]

    def closest_point(self, xy, kinds=abi.KIND_ALL):
        xy = _xy(xy)
        n = len(xy)
        pt = np.zeros((n, 2))
        d = np.zeros(n)
        seg = np.zeros(n, dtype=np.int32)
        check(load().wostgpu_closest_point(self.h, n, _d(xy), kinds, _d(pt), _d(d),
                                            seg.ctypes.data_as(C.POINTER(C.c_int32))))
        return pt, d, seg

    def closest_silhouette(self, xy):
        xy = _xy(xy)
        d = np.zeros(len(xy))
        check(load().wostgpu_closest_silhouette(self.h, len(xy), _d(xy), _d(d)))
        return d

    def ray_first_hit(self, origin, direction, t_max, kinds=abi.KIND_ALL, exclude=None):
        o = _xy(origin)
        dr = _xy(direction)
        n = len(o)
        tm = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)))
        ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.int32)
        t = np.zeros(n)
        pt = np.zeros((n, 2))
        nrm = np.zeros((n, 2))
        seg = np.zeros(n, dtype=np.int32)
        kind = np.zeros(n, dtype=np.int32)
        I = C.POINTER(C.c_int32)
        check(load().wostgpu_ray_first_hit(
            self.h, n, _d(o), _d(dr), _d(tm), kinds,
            None if ex is None else ex.ctypes.data_as(I), _d(t), _d(pt), _d(nrm),
            seg.ctypes.data_as(I), kind.ctypes.data_as(I)))
        return t, pt, nrm, seg, kind

    def star_radius(self, xy, r_min):
        xy = _xy(xy)
        r = np.zeros(len(xy))
        check(load().wostgpu_star_radius(self.h, len(xy), _d(xy), r_min, _d(r)))
        return r


class GuidingField:
    """wost::GuidingField (guide_field.hpp:37): grid + MLP on the device."""

    def __init__(self, cfg: abi.FieldConfig, bbox, seed, device=None):
        init(device)
        self.cfg = cfg
        self.bbox = tuple(bbox)
        h = C.c_void_p()
        check(load().wostgpu_field_create(C.byref(cfg), (C.c_double * 4)(*bbox), seed, C.byref(h)))
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
        return (2 + self.cfg.mixture_dim) * self.cfg.mixture_k + 1

    def params(self):
        p = np.zeros(self.n_params, dtype=np.float32)
        check(load().wostgpu_field_get_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)),
                                              None, None, None))
        return p

    def state(self):
        p = np.zeros(self.n_params, dtype=np.float32)
        m = np.zeros(self.n_params)
        v = np.zeros(self.n_params)
        steps = C.c_int64()
        check(load().wostgpu_field_get_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)),
                                              _d(m), _d(v), C.byref(steps)))
        return p, m, v, steps.value

    def set_params(self, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        check(load().wostgpu_field_set_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)),
                                              None, None, -1))

    def set_state(self, p, m, v, steps):
        p = np.ascontiguousarray(p, dtype=np.float32)
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        check(load().wostgpu_field_set_state(self.h, p.ctypes.data_as(C.POINTER(C.c_float)),
                                              _d(m), _d(v), steps))

    def get_param(self, i):
        """GuidingField::get_param (guide_field.hpp:73-77)."""
        out = np.zeros(1, dtype=np.float32)
        check(load().wostgpu_field_get_params(self.h, int(i), 1, out.ctypes.data_as(C.POINTER(C.c_float))))
        return float(out[0])

    def set_param(self, i, value):
        """GuidingField::set_param (guide_field.hpp:73-77)."""
        v = np.array([value], dtype=np.float32)
        check(load().wostgpu_field_set_params(self.h, int(i), 1, v.ctypes.data_as(C.POINTER(C.c_float))))

    def backward(self, xy, d_out, grad=None):
        """eval_with_tape + backward (guide_field.cpp:223-243, 258-315) for
        every point: grad += sum_i J(x_i)^T d_out[i] (fp64); returns grad."""
        xy = _xy(xy)
        d_out = np.ascontiguousarray(d_out, dtype=np.float64).reshape(len(xy), self.output_dim)
        g = np.zeros(self.n_params) if grad is None else grad
        assert g.dtype == np.float64 and g.shape == (self.n_params,) and g.flags.c_contiguous
        check(load().wostgpu_field_backward(self.h, len(xy), _d(xy), _d(d_out), _d(g)))
        return g

    def adam_step(self, grad, lr, beta1, beta2, eps):
        """GuidingField::adam_step (guide_field.cpp:317-331); zeroes grad."""
        assert grad.dtype == np.float64 and grad.shape == (self.n_params,) and grad.flags.c_contiguous
        check(load().wostgpu_field_adam_step(self.h, _d(grad), lr, beta1, beta2, eps))

    # WGF1 checkpoints, byte-compatible with GuidingField::save / load
    # (guide_field.cpp:333-411); see include/wostgpu.hpp for the layout
    def save(self, path):
        p, m, v, steps = self.state()
        c = self.cfg
        with open(path, "wb") as f:
            f.write(b"WGF1")
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
    def load(cls, path, device=None):
        with open(path, "rb") as f:
            data = f.read()
        if data[:4] != b"WGF1":
            raise ValueError("guiding field checkpoint: bad magic")
        off = 4
        u32 = lambda k: np.frombuffer(data, "<u4", k, off)  # noqa: E731
        ver, nl = u32(2)
        if ver != 1:
            raise ValueError("guiding field checkpoint: unknown version")
        off += 8
        res = [int(r) for r in u32(nl)]
        off += 4 * int(nl)
        feat, hid, k, dim = (int(x) for x in u32(4))
        off += 16
        bbox = tuple(float(x) for x in np.frombuffer(data, "<f8", 4, off))
        off += 32
        steps = int(np.frombuffer(data, "<i8", 1, off)[0])
        off += 8
        n = int(np.frombuffer(data, "<u8", 1, off)[0])
        off += 8
        field = cls(abi.field_config(tuple(res), features=feat, hidden=hid, mixture_k=k, mixture_dim=dim),
                    bbox, 0, device)
        if n != field.n_params:
            raise ValueError("guiding field checkpoint: size mismatch")
        if len(data) < off + n * 20:
            raise ValueError("guiding field checkpoint: truncated")
        p = np.frombuffer(data, "<f4", n, off)
        m = np.frombuffer(data, "<f8", n, off + 4 * n)
        v = np.frombuffer(data, "<f8", n, off + 12 * n)
        field.set_state(p, m, v, steps)
        return field

    def check_pack(self):
        """Bytes in which the Adam-maintained split-fp16 weight blob of the
        tensor-core kernels differs from a fresh pack (-1: no blob yet)."""
        m = C.c_int64()
        check(load().wostgpu_field_check_pack(self.h, C.byref(m)))
        return m.value

    def eval_batch(self, xy, mlp=MLP_EXACT):
        xy = _xy(xy)
        out = np.zeros((len(xy), self.output_dim))
        check(load().wostgpu_field_eval_batch(self.h, len(xy), _d(xy), _d(out), mlp))
        return out


def normalize_params(raw, k, dim=2):
    """normalize_params(unpack_params(raw)) on device (sphdist.cpp:287-310)."""
    raw = np.ascontiguousarray(raw, dtype=np.float64)
    out = np.zeros(raw.shape[0], dtype=abi.MIXTURE_DTYPE)
    check(load().wostgpu_normalize_params(raw.shape[0], _d(raw), k, dim,
                                           C.c_void_p(out.ctypes.data)))
    return out


def mixture32_pdf(raw, nu):
    """Tensor-core walk path's fp32 mixture math (diagnostic): decode each raw
    row (33 floats, K = 8) and evaluate the mixture pdf at the unit direction
    nu[i]; returns (pdf [n], c [n])."""
    raw = np.ascontiguousarray(raw, dtype=np.float32)
    nu = np.ascontiguousarray(nu, dtype=np.float64)
    out = np.zeros((raw.shape[0], 2))
    check(load().wostgpu_mixture32_pdf(raw.shape[0], raw.ctypes.data_as(C.POINTER(C.c_float)), _d(nu),
                                       _d(out)))
    return out[:, 0], out[:, 1]


def mixture32_sample(raw, n, seed):
    """n directions drawn by the tensor-core walk path's sampler from the
    single mixture `raw` (33 floats), sample i on PCG32 stream (seed, i)."""
    raw = np.ascontiguousarray(raw, dtype=np.float32).reshape(33)
    out = np.zeros((n, 2))
    check(load().wostgpu_mixture32_sample(raw.ctypes.data_as(C.POINTER(C.c_float)), n, seed, _d(out)))
    return out


class Solver:
    """StepContext + SolveScratch + the Engine's record/training state
    (wost.hpp:33-51, solver.cpp:53-105) resident on one GPU."""

    def __init__(self, accel: Accel, field: GuidingField | None, cfg: abi.SolverConfig,
                 mlp=MLP_TENSOR):
        self.accel, self.field, self.cfg = accel, field, cfg
        h = C.c_void_p()
        check(load().wostgpu_solver_create(accel.h, field.h if field else None, C.byref(cfg),
                                            C.byref(h)))
        self.h = h
        self.n_points = 0
        self.set_mlp(mlp)

    def __del__(self):
        if getattr(self, "h", None):
            load().wostgpu_solver_destroy(self.h)
            self.h = None

    def set_mlp(self, mlp):
        check(load().wostgpu_solver_set_mlp(self.h, mlp))

    def set_points(self, xy, global_offset=0):
        xy = _xy(xy)
        self.n_points = len(xy)
        check(load().wostgpu_solver_set_points(self.h, len(xy), _d(xy), global_offset))

    def stats(self):
        st = np.zeros(self.n_points, dtype=abi.POINT_STATS_DTYPE)
        check(load().wostgpu_solver_get_stats(self.h, C.c_void_p(st.ctypes.data)))
        return st

    def set_stats(self, st):
        st = np.ascontiguousarray(st, dtype=abi.POINT_STATS_DTYPE)
        check(load().wostgpu_solver_set_stats(self.h, C.c_void_p(st.ctypes.data)))

    def solve_rounds(self, seed, wpp_first, n_rounds, collect=False):
        check(load().wostgpu_solve_rounds(self.h, seed, wpp_first, n_rounds, int(collect)))

    def walks(self):
        """estimate / escaped / steps of every point in the last round."""
        n = self.n_points
        est = np.zeros(n)
        esc = np.zeros(n, dtype=np.int32)
        steps = np.zeros(n, dtype=np.int32)
        I = C.POINTER(C.c_int32)
        check(load().wostgpu_fetch_walks(self.h, _d(est), esc.ctypes.data_as(I),
                                          steps.ctypes.data_as(I)))
        return est, esc, steps

    def records(self):
        n = C.c_int64()
        check(load().wostgpu_fetch_records(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=abi.GUIDE_RECORD_DTYPE)
        check(load().wostgpu_fetch_records(self.h, C.c_void_p(out.ctypes.data), n.value,
                                            C.byref(n)))
        return out[: n.value]

    def counters(self):
        v = [C.c_int64() for _ in range(4)]
        check(load().wostgpu_solver_counters(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("walks", "steps", "escaped", "records"), (x.value for x in v)))

    def timing(self):
        w, t = C.c_double(), C.c_double()
        check(load().wostgpu_solver_timing(self.h, C.byref(w), C.byref(t)))
        return w.value, t.value

    def train_round(self, cfg: abi.TrainConfig, rnd):
        st = abi.TrainStats()
        check(load().wostgpu_train_round(self.h, C.byref(cfg), rnd, C.byref(st)))
        return st

    def train_batch(self, records, cfg: abi.TrainConfig, rnd):
        recs = np.ascontiguousarray(records, dtype=abi.GUIDE_RECORD_DTYPE)
        st = abi.TrainStats()
        check(load().wostgpu_train_batch(self.h, C.c_void_p(recs.ctypes.data), len(recs),
                                          C.byref(cfg), rnd, C.byref(st)))
        return st

    def field_grad(self, records, cfg: abi.TrainConfig):
        recs = np.ascontiguousarray(records, dtype=abi.GUIDE_RECORD_DTYPE)
        g = np.zeros(self.field.n_params)
        check(load().wostgpu_field_grad(self.h, C.c_void_p(recs.ctypes.data), len(recs),
                                         C.byref(cfg), _d(g)))
        return g

    # split-phase training round (wostgpu.h): the library's NCCL round with
    # the two allreduces (usable count, gradient sums) done by the caller
    def train_prepare(self, cfg: abi.TrainConfig):
        """Targets and validity of the last collecting round's records; returns
        this rank's usable record count."""
        u = C.c_int64()
        check(load().wostgpu_train_prepare(self.h, C.byref(cfg), C.byref(u)))
        return u.value

    def train_select(self, cfg: abi.TrainConfig, usable_global):
        """The round's training set from the global usable count; returns the
        number of minibatches."""
        nmb = C.c_int32()
        check(load().wostgpu_train_select(self.h, C.byref(cfg), int(usable_global), C.byref(nmb)))
        return nmb.value

    def train_minibatch_grad(self, cfg: abi.TrainConfig, b):
        """This rank's gradient sum of minibatch b (records pre-scaled by
        1 / minibatch); the last entry is the record count."""
        g = np.zeros(self.field.n_params + 1, dtype=np.float32)
        check(load().wostgpu_train_minibatch_grad(self.h, C.byref(cfg), b,
                                                   g.ctypes.data_as(C.POINTER(C.c_float))))
        return g

    def train_apply(self, cfg: abi.TrainConfig, grad_sum):
        """One Adam step on a (globally summed) train_minibatch_grad buffer."""
        g = np.ascontiguousarray(grad_sum, dtype=np.float32)
        assert g.shape == (self.field.n_params + 1,)
        check(load().wostgpu_train_apply(self.h, C.byref(cfg), g.ctypes.data_as(C.POINTER(C.c_float))))

    def run(self, seed, wpp, train_until=256, train_cfg: abi.TrainConfig | None = None):
        """Engine loop natively (wostgpu_run): returns (TrainStats, device ms)."""
        st = abi.TrainStats()
        ms = C.c_double()
        check(load().wostgpu_run(self.h, seed, wpp, train_until,
                                  C.byref(train_cfg) if train_cfg is not None else None,
                                  C.byref(st), C.byref(ms)))
        return st, ms.value

    def run_profile(self):
        w, t = C.c_double(), C.c_double()
        v = [C.c_int64() for _ in range(4)]
        check(load().wostgpu_run_profile(self.h, C.byref(w), C.byref(t), *[C.byref(x) for x in v]))
        out = dict(zip(("walks", "steps", "escaped", "train_steps"), (x.value for x in v)))
        out["walk_ms"], out["train_ms"] = w.value, t.value
        return out

    def reserve_records(self, n):
        """Record arena of at least n records per collecting round (a round
        that overflows the arena fails its call instead of training on a
        short-walk-biased subset)."""
        check(load().wostgpu_solver_reserve_records(self.h, int(n)))

    def attach_comm(self, unique_id: bytes, nranks, rank):
        check(load().wostgpu_solver_attach_comm(self.h, unique_id, nranks, rank))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().wostgpu_comm_unique_id(buf))
    return buf.raw


def solve_batch(solver: Solver, points, stats, seed, wpp_index, collect_records=False):
    """Drop-in solve_batch (wost.hpp:160-163): updates `stats` in place and
    returns the round's records when collect_records."""
    xy = _xy(points)
    st = np.ascontiguousarray(stats, dtype=abi.POINT_STATS_DTYPE)
    check(load().wostgpu_solve_batch(solver.h, len(xy), _d(xy), C.c_void_p(st.ctypes.data), seed,
                                      wpp_index, int(collect_records)))
    solver.n_points = len(xy)
    stats[...] = st
    return solver.records() if collect_records else None
