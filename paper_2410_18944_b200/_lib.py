"""Loads the in-tree CUDA library (libwostgpu.so) and declares its C-ABI.

There is deliberately no fallback: if the shared object is missing or no
sm_100 device is visible, every entry point raises WostGpuError.
"""
import ctypes as C
import os

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WOSTGPU_LIB") or os.path.join(_HERE, "libwostgpu.so")  # override: A/B builds

D = C.POINTER(C.c_double)
F32 = C.POINTER(C.c_float)
I32 = C.POINTER(C.c_int32)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p


class WostGpuError(RuntimeError):
    """Raised for every non-zero status of the C-ABI."""

    def __init__(self, code, msg):
        super().__init__(f"wostgpu error {code}: {msg}")
        self.code = code


class SceneError(WostGpuError):
    """wost::SceneError (proj/include/wost/scene.hpp:12)."""


class InvalidArgument(WostGpuError, ValueError):
    """std::invalid_argument in the reference."""


_SIGS = {
    "wostgpu_last_error": (C.c_char_p, []),
    "wostgpu_init": (C.c_int, [C.c_int]),
    "wostgpu_device_info": (C.c_int, [C.POINTER(C.c_int)] * 3),
    "wostgpu_kernel_launches": (C.c_int64, []),
    "wostgpu_scene_create": (C.c_int, [D, I32, I32, C.c_int32, C.POINTER(abi.ValueSpec), C.c_int32,
                                       C.POINTER(abi.ValueSpec), D, C.c_double, C.POINTER(VP)]),
    "wostgpu_scene_destroy": (C.c_int, [VP]),
    "wostgpu_scene_info": (C.c_int, [VP, D, I32, D]),
    "wostgpu_closest_point": (C.c_int, [VP, C.c_int64, D, C.c_uint32, D, D, I32]),
    "wostgpu_closest_silhouette": (C.c_int, [VP, C.c_int64, D, D]),
    "wostgpu_ray_first_hit": (C.c_int, [VP, C.c_int64, D, D, D, C.c_uint32, I32, D, D, D, I32, I32]),
    "wostgpu_star_radius": (C.c_int, [VP, C.c_int64, D, C.c_double, D]),
    "wostgpu_field_create": (C.c_int, [C.POINTER(abi.FieldConfig), D, C.c_uint64, C.POINTER(VP)]),
    "wostgpu_field_destroy": (C.c_int, [VP]),
    "wostgpu_field_param_count": (C.c_int, [VP, I64]),
    "wostgpu_field_get_state": (C.c_int, [VP, F32, D, D, I64]),
    "wostgpu_field_set_state": (C.c_int, [VP, F32, D, D, C.c_int64]),
    "wostgpu_field_eval_batch": (C.c_int, [VP, C.c_int64, D, D, C.c_int]),
    "wostgpu_normalize_params": (C.c_int, [C.c_int64, D, C.c_int32, C.c_int32, VP]),
    "wostgpu_mixture32_pdf": (C.c_int, [C.c_int64, F32, D, D]),
    "wostgpu_field_check_pack": (C.c_int, [VP, I64]),
    "wostgpu_mixture32_sample": (C.c_int, [F32, C.c_int64, C.c_uint64, D]),
    "wostgpu_mixture3f_pdf": (C.c_int, [C.c_int64, F32, D, D]),
    "wostgpu_solver_create": (C.c_int, [VP, VP, C.POINTER(abi.SolverConfig), C.POINTER(VP)]),
    "wostgpu_solver_destroy": (C.c_int, [VP]),
    "wostgpu_solver_set_mlp": (C.c_int, [VP, C.c_int]),
    "wostgpu_solver_set_points": (C.c_int, [VP, C.c_int64, D, C.c_int64]),
    "wostgpu_solver_get_stats": (C.c_int, [VP, VP]),
    "wostgpu_solver_set_stats": (C.c_int, [VP, VP]),
    "wostgpu_solve_rounds": (C.c_int, [VP, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32]),
    "wostgpu_solve_batch": (C.c_int, [VP, C.c_int64, D, VP, C.c_uint64, C.c_uint64, C.c_int32]),
    "wostgpu_fetch_records": (C.c_int, [VP, VP, C.c_int64, I64]),
    "wostgpu_fetch_walks": (C.c_int, [VP, D, I32, I32]),
    "wostgpu_solver_counters": (C.c_int, [VP, I64, I64, I64, I64]),
    "wostgpu_train_round": (C.c_int, [VP, C.POINTER(abi.TrainConfig), C.c_uint64,
                                      C.POINTER(abi.TrainStats)]),
    "wostgpu_train_batch": (C.c_int, [VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), C.c_uint64,
                                      C.POINTER(abi.TrainStats)]),
    "wostgpu_field_grad": (C.c_int, [VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), D]),
    "wostgpu_field_get_params": (C.c_int, [VP, C.c_int64, C.c_int64, F32]),
    "wostgpu_field_set_params": (C.c_int, [VP, C.c_int64, C.c_int64, F32]),
    "wostgpu_field_backward": (C.c_int, [VP, C.c_int64, D, D, D]),
    "wostgpu_field_adam_step": (C.c_int, [VP, D, C.c_double, C.c_double, C.c_double, C.c_double]),
    "wostgpu_shutdown": (C.c_int, []),
    "wostgpu_solver_reserve_records": (C.c_int, [VP, C.c_int64]),
    "wostgpu_solver3_reserve_records": (C.c_int, [VP, C.c_int64]),
    "wostgpu_train_prepare": (C.c_int, [VP, C.POINTER(abi.TrainConfig), I64]),
    "wostgpu_train_select": (C.c_int, [VP, C.POINTER(abi.TrainConfig), C.c_int64, I32]),
    "wostgpu_train_minibatch_grad": (C.c_int, [VP, C.POINTER(abi.TrainConfig), C.c_int32, F32]),
    "wostgpu_train_apply": (C.c_int, [VP, C.POINTER(abi.TrainConfig), F32]),
    "wostgpu_run": (C.c_int, [VP, C.c_uint64, C.c_int32, C.c_int64, C.POINTER(abi.TrainConfig),
                              C.POINTER(abi.TrainStats), D]),
    "wostgpu_run_profile": (C.c_int, [VP, D, D, I64, I64, I64, I64]),
    "wostgpu_comm_unique_id": (C.c_int, [C.c_char_p]),
    "wostgpu_solver_attach_comm": (C.c_int, [VP, C.c_char_p, C.c_int32, C.c_int32]),
    "wostgpu_solver_timing": (C.c_int, [VP, D, D]),
    # ---- 3D path (include/wostgpu3.h)
    "wostgpu_scene3_create": (C.c_int, [D, I32, I32, C.c_int32, C.POINTER(abi.Value3Spec), C.c_int32,
                                        C.POINTER(abi.Value3Spec), D, C.c_double, C.POINTER(VP)]),
    "wostgpu_scene3_destroy": (C.c_int, [VP]),
    "wostgpu_scene3_info": (C.c_int, [VP, D, I64, I64, I64]),
    "wostgpu_closest_point3": (C.c_int, [VP, C.c_int64, D, C.c_uint32, D, D, I32]),
    "wostgpu_closest_silhouette3": (C.c_int, [VP, C.c_int64, D, D]),
    "wostgpu_ray_first_hit3": (C.c_int, [VP, C.c_int64, D, D, D, C.c_uint32, I32, D, D, D, I32, I32]),
    "wostgpu_star_radius3": (C.c_int, [VP, C.c_int64, D, C.c_double, D]),
    "wostgpu_field3_create": (C.c_int, [C.POINTER(abi.FieldConfig), D, C.c_uint64, C.POINTER(VP)]),
    "wostgpu_field3_eval_batch": (C.c_int, [VP, C.c_int64, D, D, C.c_int]),
    "wostgpu_solver3_set_mlp": (C.c_int, [VP, C.c_int]),
    "wostgpu_solver3_create": (C.c_int, [VP, VP, C.POINTER(abi.SolverConfig), C.POINTER(VP)]),
    "wostgpu_solver3_destroy": (C.c_int, [VP]),
    "wostgpu_solver3_set_points": (C.c_int, [VP, C.c_int64, D, C.c_int64]),
    "wostgpu_solver3_get_stats": (C.c_int, [VP, VP]),
    "wostgpu_solver3_solve_rounds": (C.c_int, [VP, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32]),
    "wostgpu_solver3_fetch_walks": (C.c_int, [VP, D, I32, I32]),
    "wostgpu_solver3_fetch_records": (C.c_int, [VP, VP, C.c_int64, I64]),
    "wostgpu_solver3_counters": (C.c_int, [VP, I64, I64, I64, I64]),
    "wostgpu_solver3_train_round": (C.c_int, [VP, C.POINTER(abi.TrainConfig), C.c_uint64,
                                              C.POINTER(abi.TrainStats)]),
    "wostgpu_solver3_field_grad": (C.c_int, [VP, VP, C.c_int64, C.POINTER(abi.TrainConfig), D]),
    "wostgpu_solver3_run": (C.c_int, [VP, C.c_uint64, C.c_int32, C.c_int64, C.POINTER(abi.TrainConfig),
                                      C.POINTER(abi.TrainStats), D]),
    "wostgpu_solver3_run_profile": (C.c_int, [VP, D, D, I64, I64, I64, I64]),
    "wostgpu_solver3_attach_comm": (C.c_int, [VP, C.c_char_p, C.c_int32, C.c_int32]),
}

EXPORTED_SYMBOLS = sorted(_SIGS)

_lib = None


def load(path=None):
    """Load (once) and return the CDLL. Raises WostGpuError when missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise WostGpuError(abi.WG_ERR_NOT_BUILT,
                           f"{path} is missing: run `make` (or __graft_entry__.build())")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc != 0:
        msg = load().wostgpu_last_error().decode()
        if rc == abi.WG_ERR_SCENE:
            raise SceneError(rc, msg)
        if rc == abi.WG_ERR_INVALID:
            raise InvalidArgument(rc, msg)
        raise WostGpuError(rc, msg)


_inited = {}


def init(device=None):
    """Bind this process to a GPU (LOCAL_RANK by default)."""
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    if _inited.get("device") == device:
        return
    check(load().wostgpu_init(device))
    _inited["device"] = device


def kernel_launches():
    return int(load().wostgpu_kernel_launches())
