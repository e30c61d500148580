"""ctypes binding of libtacsl_b200.so (include/tacsl_b200.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.  A
missing library, a missing symbol or a non-B200 device raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "libtacsl_b200.so"

c_int, c_int64, c_double, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
c_char_p = ctypes.c_char_p
P = c_void_p  # every data pointer crosses as an opaque address


class Penalty(ctypes.Structure):
    _fields_ = [("k_n", c_double), ("k_d", c_double), ("k_t", c_double), ("mu", c_double)]


class AugmentCfg(ctypes.Structure):
    _fields_ = [("shift_px", c_double), ("zoom_lo", c_double), ("zoom_hi", c_double), ("brightness", c_double),
                ("contrast_lo", c_double), ("contrast_hi", c_double), ("saturation_lo", c_double),
                ("saturation_hi", c_double), ("hue", c_double), ("channel_permutation", ctypes.c_int32),
                ("step_brightness", c_double), ("step_contrast_lo", c_double), ("step_contrast_hi", c_double),
                ("step_saturation_lo", c_double), ("step_saturation_hi", c_double), ("step_hue", c_double),
                ("seed", ctypes.c_uint64)]


# name -> (restype, argtypes); mirrors include/tacsl_b200.h one for one
SIGNATURES = {
    "tacsl_abi_version": (c_int, []),
    "tacsl_last_error": (c_char_p, []),
    "tacsl_device_supported": (c_int, [c_int]),
    "tacsl_lut_create": (c_int, [P, c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
    "tacsl_lut_destroy": (None, [c_void_p]),
    "tacsl_depth_to_rgb": (c_int, [c_void_p, P, c_int64, c_int, c_int, P, P, c_void_p]),
    "tacsl_to_uint8": (c_int, [P, c_int64, P, c_void_p]),
    "tacsl_to_uint8_f64": (c_int, [P, c_int64, P, c_void_p]),
    "tacsl_f64_to_f32": (c_int, [P, c_int64, P, c_void_p]),
    "tacsl_f32_to_f64": (c_int, [P, c_int64, P, c_void_p]),
    "tacsl_frame_digest": (c_int, [P, c_int64, c_int64, P, c_void_p]),
    "tacsl_relative_penetration_rate": (c_int, [P, P, P, c_int64, c_int, P, P, c_void_p]),
    "tacsl_rgb_pyramid_supported": (c_int, [c_int, c_int, c_int, c_int]),
    "tacsl_rgb_pyramid": (c_int, [P, c_int, P, c_int64, c_int, c_int, P, c_int, P, c_void_p]),
    "tacsl_sdf_create": (c_int, [c_int, P, P, P, P, c_double, ctypes.POINTER(c_void_p)]),
    "tacsl_sdf_destroy": (None, [c_void_p]),
    "tacsl_query_sdf": (c_int, [c_void_p, P, c_int64, P, P, P, c_void_p]),
    "tacsl_penalty_forces": (c_int, [P, P, P, P, c_int64, Penalty, P, P, c_void_p]),
    "tacsl_force_field": (c_int, [c_void_p, P, c_int, c_int, P, c_int64, P, c_int64, c_int64, c_int,
                                  Penalty, c_int, P, P, P, P, P, P, c_void_p]),
    "tacsl_tactile_image_obs": (c_int, [c_void_p, P, c_int64, c_int, c_int, c_int, P, P, c_void_p]),
    "tacsl_augment_params": (c_int, [ctypes.POINTER(AugmentCfg), P, P, c_int64, P, c_void_p]),
    "tacsl_augment": (c_int, [P, c_int64, c_int, c_int, P, c_int, P, P, c_void_p]),
    "tacsl_separable_filter": (c_int, [P, c_int64, c_int, c_int, P, c_int, c_int, P, c_void_p]),
    "tacsl_sensor_step": (c_int, [c_void_p, P, c_int64, c_int, c_int, P, c_void_p, P, c_int, c_int, P, c_int64, P,
                                  c_int64, c_int64, c_int, Penalty, P, P, P, P, c_void_p]),
    "tacsl_net_wrench": (c_int, [P, P, P, c_int64, c_int, c_int, P, P, c_void_p]),
    "tacsl_binned_lut_create": (c_int, [c_int, P, c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
    "tacsl_binned_lut_destroy": (None, [c_void_p]),
    "tacsl_depth_to_rgb_binned": (c_int, [c_void_p, P, c_int64, c_int, c_int, P, P, c_void_p]),
    "tacsl_render_depth": (c_int, [c_void_p, P, P, c_int, c_int, P, c_double, c_double, c_double, c_int, P,
                                   c_int64, P, P, c_void_p]),
    "tacsl_env_render_params": (c_int, [c_void_p, P, c_int64, c_int, P, c_void_p]),
}

ABI_VERSION = 1

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; RuntimeError if unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2408_06506_b200.build` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError -> missing export
            fn.restype = res
            fn.argtypes = args
        if lib.tacsl_abi_version() != ABI_VERSION:
            raise RuntimeError("libtacsl_b200.so ABI version mismatch")
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().tacsl_last_error()
    return msg.decode() if msg else ""


_CODES = {
    1: ValueError,
    2: errors.DimensionMismatch,
    3: errors.LutResolutionMismatch,
    4: errors.InvalidQuery,
    5: RuntimeError,
    6: RuntimeError,
}


def check(rc: int) -> None:
    """Map a tacsl_status_t to the reference's exception types."""
    if rc == 0:
        return
    raise _CODES.get(rc, RuntimeError)(last_error() or f"tacsl error {rc}")


def penalty(params) -> Penalty:
    return Penalty(float(params.k_n), float(params.k_d), float(params.k_t), float(params.mu))
