"""ctypes bindings for the CPU oracle (oracle/liboracle.so, prefix orc_) and the
reference library itself (oracle/_ref/libwost_ref.so, prefix ref_).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py. Both libraries expose the same ABI
(oracle/oracle_abi.h), so `Oracle("orc")` and `Oracle("ref")` are drop-in
replacements of each other.
"""
import ctypes as C
import os

import numpy as np

from paper_2410_18944_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libwost_ref.so")
REF_FAST_SO = os.path.join(ROOT, "oracle", "_ref", "libwost_ref_fast.so")

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
F32 = C.POINTER(C.c_float)
VP = C.c_void_p


def _sig(lib, p):
    def s(name, res, *args):
        f = getattr(lib, f"{p}_{name}")
        f.restype = res
        f.argtypes = list(args)
    s("last_error", C.c_char_p)
    s("scene_create", VP, D, I32, I32, C.c_int32, C.POINTER(abi.ValueSpec), C.c_int32,
      C.POINTER(abi.ValueSpec), D, C.c_double)
    s("scene_destroy", None, VP)
    s("t_epsilon", C.c_double, VP)
    s("has_neumann_flux", C.c_int32, VP)
    s("closest_point", C.c_int, VP, C.c_int64, D, C.c_uint32, D, D, I32)
    s("closest_silhouette", C.c_int, VP, C.c_int64, D, D)
    s("ray_first_hit", C.c_int, VP, C.c_int64, D, D, D, C.c_uint32, I32, D, D, D, I32, I32)
    s("star_radius", C.c_int, VP, C.c_int64, D, C.c_double, D)
    s("bessel_i0", C.c_double, C.c_double)
    s("log_bessel_i0", C.c_double, C.c_double)
    s("bessel_i1_over_i0", C.c_double, C.c_double)
    s("normalize_params", None, C.c_int64, D, C.c_int32, C.c_int32, VP)
    s("mixture_pdf", C.c_double, VP, D)
    s("mis_pdf", C.c_double, VP, D, D, C.c_int32)
    s("field_create", VP, C.POINTER(abi.FieldConfig), D, C.c_uint64)
    s("field_destroy", None, VP)
    s("field_param_count", C.c_int64, VP)
    s("field_get_params", None, VP, F32)
    s("field_set_params", None, VP, F32)
    s("field_eval_batch", None, VP, C.c_int64, D, D)
    s("walks", C.c_int, VP, VP, C.POINTER(abi.SolverConfig), C.c_int64, D, I64, C.c_uint64,
      C.c_uint64, D, I32, I32)
    s("solve_batch", C.c_int, VP, VP, C.POINTER(abi.SolverConfig), C.c_int64, D, VP, C.c_uint64,
      C.c_uint64, C.c_int32, C.POINTER(VP), I64)
    s("free", None, VP)
    s("train_batch", C.c_int, VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), C.c_uint64,
      C.POINTER(abi.TrainStats))
    s("field_grad", C.c_int, VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), D)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """Same call surface for the restatement ("orc") and the reference ("ref")."""

    def __init__(self, which="orc", path=None):
        self.p = which
        path = path or (ORACLE_SO if which == "orc" else REF_SO)
        self.lib = C.CDLL(path)
        _sig(self.lib, which)
        if which == "ref":
            f = self.lib.ref_run_solve
            f.restype = C.c_int
            f.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                          C.c_uint64, VP, D, D, D]
            f = self.lib.ref_preset
            f.restype = C.c_int
            f.argtypes = [C.c_char_p, D, I32, I32, D, D, D]
            self.lib.ref_strip_vlin_solution.restype = C.c_double
            self.lib.ref_strip_vlin_solution.argtypes = [C.c_double, C.c_double]
            # WGF1 checkpoints through the reference's GuidingField::save / load
            if hasattr(self.lib, "ref_field_save"):
                self.lib.ref_field_save.restype = C.c_int
                self.lib.ref_field_save.argtypes = [VP, C.c_char_p]
                self.lib.ref_field_load.restype = VP
                self.lib.ref_field_load.argtypes = [C.c_char_p]
                self.lib.ref_field_adam_steps.restype = C.c_int64
                self.lib.ref_field_adam_steps.argtypes = [VP]
            if hasattr(self.lib, "ref_field_backward"):
                self.lib.ref_field_backward.restype = None
                self.lib.ref_field_backward.argtypes = [VP, C.c_int64, D, D, D]
            if hasattr(self.lib, "ref_field_adam_step"):
                self.lib.ref_field_adam_step.restype = None
                self.lib.ref_field_adam_step.argtypes = [VP, D, C.c_double, C.c_double, C.c_double,
                                                         C.c_double]

    def fn(self, name):
        return getattr(self.lib, f"{self.p}_{name}")

    def check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.fn("last_error")().decode())

    # ---- scenes
    def scene(self, sc):
        h = self.fn("scene_create")(*sc.c_args())
        if not h:
            raise OracleError(abi.WG_ERR_SCENE, self.fn("last_error")().decode())
        return h

    def scene_destroy(self, h):
        self.fn("scene_destroy")(h)

    # ---- geometry
    def closest_point(self, h, xy, kinds):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        n = len(xy)
        pt = np.zeros((n, 2))
        d = np.zeros(n)
        seg = np.zeros(n, dtype=np.int32)
        self.check(self.fn("closest_point")(h, n, abi.ptr(xy), kinds, abi.ptr(pt), abi.ptr(d),
                                             abi.ptr(seg, C.c_int32)))
        return pt, d, seg

    def closest_silhouette(self, h, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        d = np.zeros(len(xy))
        self.check(self.fn("closest_silhouette")(h, len(xy), abi.ptr(xy), abi.ptr(d)))
        return d

    def ray_first_hit(self, h, o, d, tmax, kinds, exclude=None):
        o = np.ascontiguousarray(o, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        n = len(o)
        tmax = np.ascontiguousarray(np.broadcast_to(tmax, (n,)), dtype=np.float64)
        ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.int32)
        t = np.zeros(n)
        pt = np.zeros((n, 2))
        nrm = np.zeros((n, 2))
        seg = np.zeros(n, dtype=np.int32)
        kind = np.zeros(n, dtype=np.int32)
        self.check(self.fn("ray_first_hit")(h, n, abi.ptr(o), abi.ptr(d), abi.ptr(tmax), kinds,
                                             abi.ptr(ex, C.c_int32), abi.ptr(t), abi.ptr(pt),
                                             abi.ptr(nrm), abi.ptr(seg, C.c_int32),
                                             abi.ptr(kind, C.c_int32)))
        return t, pt, nrm, seg, kind

    def star_radius(self, h, xy, r_min):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        r = np.zeros(len(xy))
        self.check(self.fn("star_radius")(h, len(xy), abi.ptr(xy), r_min, abi.ptr(r)))
        return r

    # ---- sphdist
    def normalize(self, raw, k, dim=2):
        raw = np.ascontiguousarray(raw, dtype=np.float64)
        n = raw.shape[0]
        out = np.zeros(n, dtype=abi.MIXTURE_DTYPE)
        self.fn("normalize_params")(n, abi.ptr(raw), k, dim, abi.vptr(out))
        return out

    # ---- field
    def field(self, cfg, bbox, seed):
        h = self.fn("field_create")(C.byref(cfg), (C.c_double * 4)(*bbox), seed)
        if not h:
            raise OracleError(abi.WG_ERR_INVALID, self.fn("last_error")().decode())
        return h

    def field_params(self, f):
        n = self.fn("field_param_count")(f)
        out = np.zeros(n, dtype=np.float32)
        self.fn("field_get_params")(f, abi.ptr(out, C.c_float))
        return out

    def field_set_params(self, f, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        self.fn("field_set_params")(f, abi.ptr(p, C.c_float))

    def field_eval(self, f, xy, od):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.zeros((len(xy), od))
        self.fn("field_eval_batch")(f, len(xy), abi.ptr(xy), abi.ptr(out))
        return out

    # ---- walks
    def walks(self, h, field, cfg, xy, seed, wpp, point_index=None, records=False):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        n = len(xy)
        pi = None if point_index is None else np.ascontiguousarray(point_index, dtype=np.int64)
        est = np.zeros(n)
        esc = np.zeros(n, dtype=np.int32)
        nrec = np.zeros(n, dtype=np.int32) if records else None
        self.check(self.fn("walks")(h, field, C.byref(cfg), n, abi.ptr(xy), abi.ptr(pi, C.c_int64),
                                     seed, wpp, abi.ptr(est), abi.ptr(esc, C.c_int32),
                                     abi.ptr(nrec, C.c_int32)))
        return est, esc, nrec

    def solve_batch(self, h, field, cfg, xy, stats, seed, wpp, collect=False):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        recp = VP()
        nrec = C.c_int64(0)
        self.check(self.fn("solve_batch")(h, field, C.byref(cfg), len(xy), abi.ptr(xy),
                                           abi.vptr(stats), seed, wpp, int(collect),
                                           C.byref(recp) if collect else None,
                                           C.byref(nrec) if collect else None))
        if not collect:
            return None
        n = nrec.value
        buf = (C.c_char * (n * abi.GUIDE_RECORD_DTYPE.itemsize)).from_address(recp.value)
        recs = np.frombuffer(bytes(buf), dtype=abi.GUIDE_RECORD_DTYPE).copy()
        self.fn("free")(recp)
        return recs

    def train_batch(self, f, recs, cfg, rnd):
        recs = np.ascontiguousarray(recs, dtype=abi.GUIDE_RECORD_DTYPE)
        st = abi.TrainStats()
        self.check(self.fn("train_batch")(f, abi.vptr(recs), len(recs), C.byref(cfg), rnd,
                                           C.byref(st)))
        return st

    def field_grad(self, f, recs, cfg):
        recs = np.ascontiguousarray(recs, dtype=abi.GUIDE_RECORD_DTYPE)
        g = np.zeros(self.fn("field_param_count")(f))
        self.check(self.fn("field_grad")(f, abi.vptr(recs), len(recs), C.byref(cfg), abi.ptr(g)))
        return g


def _sig3(lib):
    def s(name, res, *args):
        f = getattr(lib, f"orc3_{name}")
        f.restype = res
        f.argtypes = list(args)
    s("scene_create", VP, D, I32, I32, C.c_int32, C.POINTER(abi.Value3Spec), C.c_int32,
      C.POINTER(abi.Value3Spec), D, C.c_double)
    s("scene_destroy", None, VP)
    s("t_epsilon", C.c_double, VP)
    s("silhouette_info", None, VP, I64, I64)
    s("closest_point", C.c_int, VP, C.c_int64, D, C.c_uint32, D, D, I32)
    s("closest_silhouette", C.c_int, VP, C.c_int64, D, D)
    s("ray_first_hit", C.c_int, VP, C.c_int64, D, D, D, C.c_uint32, I32, D, D, D, I32, I32)
    s("star_radius", C.c_int, VP, C.c_int64, D, C.c_double, D)
    s("field_create", VP, C.POINTER(abi.FieldConfig), D, C.c_uint64)
    s("field_destroy", None, VP)
    s("field_param_count", C.c_int64, VP)
    s("field_get_params", None, VP, F32)
    s("field_set_params", None, VP, F32)
    s("field_eval_batch", None, VP, C.c_int64, D, D)
    s("walks", C.c_int, VP, VP, C.POINTER(abi.SolverConfig), C.c_int64, D, I64, C.c_uint64,
      C.c_uint64, D, I32, I32)
    s("walk_records", C.c_int, VP, VP, C.POINTER(abi.SolverConfig), C.c_int64, D, I64, C.c_uint64,
      C.c_uint64, C.POINTER(VP), I64)
    s("field_grad", C.c_int, VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), D)
    s("train_batch", C.c_int, VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), C.c_uint64,
      C.POINTER(abi.TrainStats))
    s("run", C.c_int, VP, VP, C.POINTER(abi.SolverConfig), C.c_int64, D, C.c_int64, C.c_uint64,
      C.c_int32, C.c_int64, C.POINTER(abi.TrainConfig), VP)


class Oracle3:
    """The 3D contract restatement (oracle/wost3d.inc, prefix orc3_). There is
    no reference 3D code, so there is no "ref" counterpart."""

    def __init__(self, path=None):
        self.lib = C.CDLL(path or ORACLE_SO)
        _sig(self.lib, "orc")
        _sig3(self.lib)

    def fn(self, name):
        return getattr(self.lib, f"orc3_{name}")

    def check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def scene(self, sc):
        h = self.fn("scene_create")(*sc.c_args())
        if not h:
            raise OracleError(abi.WG_ERR_SCENE, self.lib.orc_last_error().decode())
        return h

    def scene_destroy(self, h):
        self.fn("scene_destroy")(h)

    def silhouette_info(self, h):
        a, c = C.c_int64(0), C.c_int64(0)
        self.fn("silhouette_info")(h, C.byref(a), C.byref(c))
        return a.value, c.value

    def closest_point(self, h, x, kinds):
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = len(x)
        pt = np.zeros((n, 3))
        d = np.zeros(n)
        tri = np.zeros(n, dtype=np.int32)
        self.check(self.fn("closest_point")(h, n, abi.ptr(x), kinds, abi.ptr(pt), abi.ptr(d),
                                             abi.ptr(tri, C.c_int32)))
        return pt, d, tri

    def closest_silhouette(self, h, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        d = np.zeros(len(x))
        self.check(self.fn("closest_silhouette")(h, len(x), abi.ptr(x), abi.ptr(d)))
        return d

    def ray_first_hit(self, h, o, d, tmax, kinds, exclude=None):
        o = np.ascontiguousarray(o, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        n = len(o)
        tmax = np.ascontiguousarray(np.broadcast_to(tmax, (n,)), dtype=np.float64)
        ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.int32)
        t = np.zeros(n)
        pt = np.zeros((n, 3))
        nrm = np.zeros((n, 3))
        tri = np.zeros(n, dtype=np.int32)
        kind = np.zeros(n, dtype=np.int32)
        self.check(self.fn("ray_first_hit")(h, n, abi.ptr(o), abi.ptr(d), abi.ptr(tmax), kinds,
                                             abi.ptr(ex, C.c_int32), abi.ptr(t), abi.ptr(pt),
                                             abi.ptr(nrm), abi.ptr(tri, C.c_int32),
                                             abi.ptr(kind, C.c_int32)))
        return t, pt, nrm, tri, kind

    def star_radius(self, h, x, r_min):
        x = np.ascontiguousarray(x, dtype=np.float64)
        r = np.zeros(len(x))
        self.check(self.fn("star_radius")(h, len(x), abi.ptr(x), r_min, abi.ptr(r)))
        return r

    def field(self, cfg, bbox, seed):
        h = self.fn("field_create")(C.byref(cfg), (C.c_double * 6)(*bbox), seed)
        if not h:
            raise OracleError(abi.WG_ERR_INVALID, self.lib.orc_last_error().decode())
        return h

    def field_destroy(self, f):
        self.fn("field_destroy")(f)

    def field_params(self, f):
        out = np.zeros(self.fn("field_param_count")(f), dtype=np.float32)
        self.fn("field_get_params")(f, abi.ptr(out, C.c_float))
        return out

    def field_set_params(self, f, p):
        p = np.ascontiguousarray(p, dtype=np.float32)
        self.fn("field_set_params")(f, abi.ptr(p, C.c_float))

    def field_eval(self, f, x, od):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((len(x), od))
        self.fn("field_eval_batch")(f, len(x), abi.ptr(x), abi.ptr(out))
        return out

    def walks(self, h, field, cfg, x, seed, wpp, point_index=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = len(x)
        pi = np.ascontiguousarray(np.arange(n) if point_index is None else point_index, dtype=np.int64)
        est = np.zeros(n)
        esc = np.zeros(n, dtype=np.int32)
        steps = np.zeros(n, dtype=np.int32)
        self.check(self.fn("walks")(h, field, C.byref(cfg), n, abi.ptr(x), abi.ptr(pi, C.c_int64),
                                     seed, wpp, abi.ptr(est), abi.ptr(esc, C.c_int32),
                                     abi.ptr(steps, C.c_int32)))
        return est, esc, steps

    def walk_records(self, h, field, cfg, x, seed, wpp, point_index=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = len(x)
        pi = np.ascontiguousarray(np.arange(n) if point_index is None else point_index, dtype=np.int64)
        recp = VP()
        nrec = C.c_int64(0)
        self.check(self.fn("walk_records")(h, field, C.byref(cfg), n, abi.ptr(x),
                                            abi.ptr(pi, C.c_int64), seed, wpp, C.byref(recp),
                                            C.byref(nrec)))
        m = nrec.value
        buf = (C.c_char * (m * abi.GUIDE_RECORD3_DTYPE.itemsize)).from_address(recp.value)
        recs = np.frombuffer(bytes(buf), dtype=abi.GUIDE_RECORD3_DTYPE).copy()
        self.lib.orc_free(recp)
        return recs

    def field_grad(self, f, recs, cfg):
        recs = np.ascontiguousarray(recs, dtype=abi.GUIDE_RECORD3_DTYPE)
        g = np.zeros(self.fn("field_param_count")(f))
        self.check(self.fn("field_grad")(f, abi.vptr(recs), len(recs), C.byref(cfg), abi.ptr(g)))
        return g

    def train_batch(self, f, recs, cfg, rnd):
        recs = np.ascontiguousarray(recs, dtype=abi.GUIDE_RECORD3_DTYPE)
        st = abi.TrainStats()
        self.check(self.fn("train_batch")(f, abi.vptr(recs), len(recs), C.byref(cfg), rnd, C.byref(st)))
        return st

    def run(self, h, field, cfg, x, seed, wpp, train_until=0, train_cfg=None, point_offset=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        st = np.zeros(len(x), dtype=abi.POINT_STATS_DTYPE)
        self.check(self.fn("run")(h, field, C.byref(cfg), len(x), abi.ptr(x), point_offset, seed, wpp,
                                   train_until, C.byref(train_cfg) if train_cfg else None,
                                   abi.vptr(st)))
        return st


def have_ref():
    return os.path.exists(REF_SO)
