"""ctypes mirrors of the plain-C structs in include/wostgpu_types.h.

These are the boundary types of the C-ABI (include/wostgpu.h). Each mirrors a
reference C++ type field for field (citations in the C header)."""
import ctypes as C

import numpy as np

WG_OK, WG_ERR_INVALID, WG_ERR_SCENE, WG_ERR_RUNTIME, WG_ERR_CUDA, WG_ERR_NOT_BUILT = range(6)
DIRICHLET, NEUMANN = 0, 1
KIND_DIRICHLET, KIND_NEUMANN, KIND_ALL = 1, 2, 3
MODE_UNIFORM, MODE_GUIDING_ONLY, MODE_FIXED_MIS, MODE_LEARNABLE_MIS = 0, 1, 2, 3
MODES = {"uniform": 0, "guiding_only": 1, "fixed_mis": 2, "learnable_mis": 3}
VALUE_ZERO, VALUE_CONSTANT, VALUE_LINEAR, VALUE_RASTER, VALUE_ANALYTIC = -1, 0, 1, 2, 3
ANALYTIC_X2_MINUS_Y2, ANALYTIC_R2_MINUS_1 = 1, 2
MAX_LEVELS = 8
MAX_MIXTURE = 16


class ValueSpec(C.Structure):
    _fields_ = [
        ("type", C.c_int32),
        ("analytic_id", C.c_int32),
        ("c0", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("raster_w", C.c_int32),
        ("raster_h", C.c_int32),
        ("raster_bbox", C.c_double * 4),
        ("raster_data", C.POINTER(C.c_double)),
    ]


class SolverConfig(C.Structure):
    _fields_ = [
        ("epsilon_shell", C.c_double),
        ("r_min", C.c_double),
        ("rr_depth", C.c_int32),
        ("mode", C.c_int32),
        ("fixed_c", C.c_double),
        ("reflect_at_neumann", C.c_int32),
        ("clamp_grazing", C.c_int32),
        ("grazing_floor", C.c_double),
        ("max_steps", C.c_int32),
        ("pad_", C.c_int32),
    ]


def solver_config(mode="uniform", epsilon_shell=0.0, r_min=0.0, rr_depth=128, fixed_c=0.5,
                  reflect=True, clamp_grazing=False, grazing_floor=1e-3, max_steps=1 << 16):
    """SolverConfig defaults of proj/include/wost/wost.hpp:20-31."""
    m = MODES[mode] if isinstance(mode, str) else int(mode)
    return SolverConfig(epsilon_shell, r_min, rr_depth, m, fixed_c, int(reflect),
                        int(clamp_grazing), grazing_floor, max_steps, 0)


class FieldConfig(C.Structure):
    _fields_ = [
        ("n_levels", C.c_int32),
        ("level_res", C.c_int32 * MAX_LEVELS),
        ("features", C.c_int32),
        ("hidden", C.c_int32),
        ("mixture_k", C.c_int32),
        ("mixture_dim", C.c_int32),
    ]


def field_config(level_res=(16, 32, 64, 128), features=4, hidden=64, mixture_k=8, mixture_dim=2):
    """FieldConfig defaults of proj/include/wost/guide_field.hpp:13-25."""
    lr = (C.c_int32 * MAX_LEVELS)(*level_res)
    return FieldConfig(len(level_res), lr, features, hidden, mixture_k, mixture_dim)


def field_param_count(cfg):
    emb = sum(r * r * cfg.features for r in cfg.level_res[: cfg.n_levels])
    i = cfg.n_levels * cfg.features
    h = cfg.hidden
    o = (2 + cfg.mixture_dim) * cfg.mixture_k + 1
    return emb + i * h + h + h * h + h + h * o + o


class Value3Spec(C.Structure):
    """wg_value3_spec (include/wostgpu_types.h): 3D Dirichlet value."""
    _fields_ = [
        ("type", C.c_int32),
        ("pad_", C.c_int32),
        ("c0", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("cz", C.c_double),
    ]


class GuideRecord3(C.Structure):
    """wg_guide_record3: GuideRecord with 3D position and normal."""
    _fields_ = [
        ("x", C.c_double * 3),
        ("nu", C.c_double * 3),
        ("target", C.c_double),
        ("pdf_mis", C.c_double),
        ("pdf_g", C.c_double),
        ("pdf_u", C.c_double),
        ("c", C.c_double),
        ("on_neumann", C.c_int32),
        ("pad_", C.c_int32),
        ("normal", C.c_double * 3),
    ]


def field_config3(level_res=(8, 16, 32, 64), features=4, hidden=64, mixture_k=8):
    """3D field: dense D^3 x F grids per level (no reference counterpart; the
    finest level is 64^3 so the 3D grid, 1.2M parameters, stays L2-resident)."""
    return field_config(level_res, features, hidden, mixture_k, 3)


def field_param_count3(cfg):
    emb = sum(r * r * r * cfg.features for r in cfg.level_res[: cfg.n_levels])
    i, h = cfg.n_levels * cfg.features, cfg.hidden
    o = (2 + cfg.mixture_dim) * cfg.mixture_k + 1
    return emb + i * h + h + h * h + h + h * o + o


class TrainConfig(C.Structure):
    _fields_ = [
        ("minibatch", C.c_int32),
        ("learn_selection", C.c_int32),
        ("max_records_per_round", C.c_int64),
        ("lr", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("e_fraction", C.c_double),
        ("reflect", C.c_int32),
        ("pad_", C.c_int32),
        ("pdf_floor", C.c_double),
        ("v_floor", C.c_double),
        ("seed", C.c_uint64),
    ]


def train_config(minibatch=1 << 14, max_records=1 << 15, lr=1e-2, beta1=0.9, beta2=0.99, eps=1e-8,
                 e_fraction=0.2, learn_selection=True, reflect=True, pdf_floor=1e-8,
                 v_floor=1e-12, seed=0):
    """TrainConfig defaults of proj/include/wost/guide_train.hpp:60-75."""
    return TrainConfig(minibatch, int(learn_selection), max_records, lr, beta1, beta2, eps,
                       e_fraction, int(reflect), 0, pdf_floor, v_floor, seed)


class TrainStats(C.Structure):
    _fields_ = [
        ("records_seen", C.c_int64),
        ("records_consumed", C.c_int64),
        ("skipped_low_pdf", C.c_int64),
        ("skipped_low_v", C.c_int64),
        ("steps", C.c_int64),
        ("mean_grad_norm", C.c_double),
        ("seconds", C.c_double),
    ]


POINT_STATS_DTYPE = np.dtype([("mean", "<f8"), ("m2", "<f8"), ("count", "<i8"), ("escaped", "<i8")])

GUIDE_RECORD_DTYPE = np.dtype([
    ("x", "<f8", 2), ("nu", "<f8", 3), ("target", "<f8"), ("pdf_mis", "<f8"), ("pdf_g", "<f8"),
    ("pdf_u", "<f8"), ("c", "<f8"), ("on_neumann", "<i4"), ("pad_", "<i4"), ("normal", "<f8", 2),
])

GUIDE_RECORD3_DTYPE = np.dtype([
    ("x", "<f8", 3), ("nu", "<f8", 3), ("target", "<f8"), ("pdf_mis", "<f8"), ("pdf_g", "<f8"),
    ("pdf_u", "<f8"), ("c", "<f8"), ("on_neumann", "<i4"), ("pad_", "<i4"), ("normal", "<f8", 3),
])

MIXTURE_DTYPE = np.dtype([
    ("mu", "<f8", (MAX_MIXTURE, 3)), ("kappa", "<f8", MAX_MIXTURE), ("lambda", "<f8", MAX_MIXTURE),
    ("log_a", "<f8", MAX_MIXTURE), ("c", "<f8"), ("k", "<i4"), ("dim", "<i4"),
])


def ptr(a, ctype=C.c_double):
    """ctypes pointer to a contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)
