"""ctypes binding of libsgmsf.so (include/sgmsf.h, include/sgmflow.h): argument marshalling only.

Every step of the method runs in the library's CUDA kernels; this module turns
Python ints / pointers into the C types of the ABI and raises on non-OK
status.  It never falls back to any other implementation: if the library is
missing or fails to load, ``load()`` raises ``SgmLibraryError``.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

LIB_PATH = _build.LIB

SGM_OK = 0
STATUS = {0: "SGM_OK", 1: "SGM_ERR_INVALID_ARGUMENT", 2: "SGM_ERR_UNSUPPORTED", 3: "SGM_ERR_CUDA",
          4: "SGM_ERR_OUT_OF_MEMORY"}
NUM_STAGES = 5

# Every symbol include/*.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "sgm_create", "sgm_destroy", "sgm_status_string", "sgm_census", "sgm_cost", "sgm_aggregate",
    "sgm_wta", "sgm_lr_check", "sgm_disparity", "sgm_combine_sceneflow", "sgm_scene_flow",
    "sgm_scene_flow_host", "sgm_set_timing", "sgm_read_timing", "sgm_stage_name",
    "sgm_launch_count", "sgm_get_geometry", "sgm_last_error_string", "sgm_debug_set_trace",
    "sgm_evaluate", "sgm_eval_rates", "sgm_scene_flow_stream", "sgm_scene_flow_stream_host",
    "sgm_get_device_error", "sgm_debug_set_flags",
    # include/sgmflow.h
    "sgm_flow_create", "sgm_flow_destroy", "sgm_flow_last_error_string", "sgm_flow_launch_count",
    "sgm_flow", "sgm_flow_field", "sgm_flow_descriptors", "sgm_flow_patch_cost",
    "sgm_flow_knn_init", "sgm_flow_sweep", "sgm_flow_consistency", "sgm_flow_set_timing",
    "sgm_flow_read_timing", "sgm_densify", "sgm_densify_scratch_bytes",
)


class SgmLibraryError(RuntimeError):
    pass


class SgmError(RuntimeError):
    def __init__(self, fn, code, lib=None):
        msg = STATUS.get(code, str(code))
        if lib is not None:
            try:
                msg += ": " + lib.sgm_status_string(code).decode()
                if code == 3:
                    err = lib.sgm_flow_last_error_string if fn.startswith(("sgm_flow", "sgm_densify")) \
                        else lib.sgm_last_error_string
                    msg += " (" + err().decode() + ")"
            except Exception:  # pragma: no cover
                pass
        super().__init__(f"{fn} failed: {msg}")
        self.code = code


class SgmParams(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("num_disp", ctypes.c_int32), ("census_w", ctypes.c_int32),
                ("census_h", ctypes.c_int32), ("p1", ctypes.c_int32), ("p2", ctypes.c_int32),
                ("lr_threshold", ctypes.c_int32), ("invalid_disp", ctypes.c_int32),
                ("bilinear_rule", ctypes.c_int32), ("max_batch", ctypes.c_int32)]


class SgmCamera(ctypes.Structure):
    _fields_ = [("f_px", ctypes.c_float), ("baseline_m", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float)]


class SgmSceneflowOut(ctypes.Structure):
    _fields_ = [("sf", ctypes.c_void_p), ("valid_sf", ctypes.c_void_p),
                ("p0", ctypes.c_void_p), ("dp", ctypes.c_void_p),
                ("valid_3d", ctypes.c_void_p), ("disp_int", ctypes.c_void_p),
                ("disp_sub", ctypes.c_void_p), ("disp_valid", ctypes.c_void_p)]


class SgmFlowParams(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("patch_radius", ctypes.c_int32), ("sweeps", ctypes.c_int32),
                ("search_radius", ctypes.c_int32), ("desc_window", ctypes.c_int32),
                ("knn", ctypes.c_int32), ("consistency_q", ctypes.c_int32),
                ("penalty", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


_lib = None


def load(path: str | None = None):
    """Load libsgmsf.so (building it first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path) or not _build.up_to_date():
        if os.path.exists(_build.NVCC):
            _build.build()
    if not os.path.exists(path):
        raise SgmLibraryError(f"{path} is missing: run `python -m paper_1801_04720_b200.build`")
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:
        raise SgmLibraryError(f"cannot load {path}: {e}") from e
    P = ctypes.c_void_p
    I32 = ctypes.c_int32
    I64 = ctypes.c_int64
    st = ctypes.c_int
    sig = {
        "sgm_create": (st, [ctypes.POINTER(SgmParams), I32, ctypes.POINTER(P)]),
        "sgm_destroy": (None, [P]),
        "sgm_status_string": (ctypes.c_char_p, [st]),
        "sgm_last_error_string": (ctypes.c_char_p, []),
        "sgm_census": (st, [P, P, I64, P, P]),
        "sgm_cost": (st, [P, P, P, I32, P, P]),
        "sgm_aggregate": (st, [P, P, P, I32, P, P]),
        "sgm_wta": (st, [P, P, P, P, P]),
        "sgm_lr_check": (st, [P, P, P, P, P, P, P, P]),
        "sgm_disparity": (st, [P, P, P, I64, P, P, P, P]),
        "sgm_combine_sceneflow": (st, [P, P, P, P, P, P, P, ctypes.POINTER(SgmCamera), P, P, P,
                                       P, P, P]),
        "sgm_scene_flow": (st, [P, I32, P, I64, P, P, ctypes.POINTER(SgmCamera),
                                ctypes.POINTER(SgmSceneflowOut), P]),
        "sgm_scene_flow_stream": (st, [P, I32, P, I64, P, P, ctypes.POINTER(SgmCamera),
                                ctypes.POINTER(SgmSceneflowOut), P]),
        "sgm_scene_flow_host": (st, [P, I32, P, P, P, ctypes.POINTER(SgmCamera),
                                     ctypes.POINTER(SgmSceneflowOut), P]),
        "sgm_scene_flow_stream_host": (st, [P, I32, P, P, P, ctypes.POINTER(SgmCamera),
                                     ctypes.POINTER(SgmSceneflowOut), P]),
        "sgm_evaluate": (st, [P, I32, P, P, P, P, P, P, P, ctypes.c_float, ctypes.c_float, P, P]),
        "sgm_eval_rates": (st, [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_double)]),
        "sgm_set_timing": (st, [P, I32]),
        "sgm_read_timing": (I32, [P, ctypes.POINTER(ctypes.c_float)]),
        "sgm_stage_name": (ctypes.c_char_p, [I32]),
        "sgm_launch_count": (I64, [P]),
        "sgm_debug_set_trace": (st, [P, P]),
        "sgm_get_device_error": (st, [P, ctypes.POINTER(I32), I32]),
        "sgm_debug_set_flags": (st, [P, I32]),
        "sgm_get_geometry": (st, [P, ctypes.POINTER(I32), ctypes.POINTER(I32),
                                  ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "sgm_flow_create": (st, [ctypes.POINTER(SgmFlowParams), I32, ctypes.POINTER(P)]),
        "sgm_flow_destroy": (None, [P]),
        "sgm_flow_last_error_string": (ctypes.c_char_p, []),
        "sgm_flow_launch_count": (I64, [P]),
        "sgm_flow": (st, [P, I32, P, P, P, P, P, P]),
        "sgm_flow_field": (st, [P, I32, P, P, ctypes.c_uint64, I32, P, P, P]),
        "sgm_flow_descriptors": (st, [P, P, I32, I32, P, P]),
        "sgm_flow_patch_cost": (st, [P, P, P, I32, I32, I32, I32, P, P, P]),
        "sgm_flow_knn_init": (st, [P, P, P, I32, I32, I32, P, P, P, P]),
        "sgm_flow_sweep": (st, [P, P, P, I32, I32, I32, I32, I32, ctypes.c_uint64, P, P, P]),
        "sgm_flow_consistency": (st, [P, P, P, P, I32, I32, P, P]),
        "sgm_flow_set_timing": (st, [P, I32]),
        "sgm_densify": (st, [I32, I32, I32, I32, P, P, P, I32, ctypes.c_float, I32, P, P, P, P, I64, P]),
        "sgm_densify_scratch_bytes": (I64, [I32, I32, I32]),
        "sgm_flow_read_timing": (I32, [P, ctypes.POINTER(ctypes.c_float)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(fn_name: str, code: int):
    if code != SGM_OK:
        raise SgmError(fn_name, code, _lib)


def call(name: str, *args):
    """Call an sgm_* function that returns sgm_status; raise on failure."""
    lib = load()
    code = getattr(lib, name)(*args)
    check(name, code)
