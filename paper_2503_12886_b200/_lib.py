"""ctypes binding of ``lib/libhs_b200.so`` (the C ABI in include/hs_api.h).

There is no fallback: if the library is missing or no CUDA device is present the
product path raises.  Status codes map to the reference's exception types
(SURVEY §8b): HS_ERR_SHAPE -> ValueError, HS_ERR_NONFINITE / HS_ERR_ZERO_QUAT ->
FloatingPointError, HS_ERR_COLOR_INIT -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HS_B200_LIB") or os.path.join(PKG, "lib", "libhs_b200.so")

HS_OK, HS_ERR_SHAPE, HS_ERR_NONFINITE, HS_ERR_ZERO_QUAT, HS_ERR_COLOR_INIT, HS_ERR_CUDA = range(6)
HS_NO_ERROR = 0xFFFFFFFFFFFFFFFF

RASTER_LOSS = 1
RASTER_IMAGE = 2
LOSS_PARTIALS_PER_TILE = 16  # hs_api.h HS_LOSS_PARTIALS_PER_TILE
RASTER_MAXW_ALL = 4
RASTER_MAXW_UNVISITED = 8
RASTER_WSUMS = 16
RASTER_WSUMS_IMAGE = 32
RASTER_ORDER_READY = 64
RASTER_DETERMINISTIC = 128
RASTER_RAW_MEAN = 256
FILL_CTA_SORT = 1                 # hs_tile_fill flags (HS_FILL_CTA_SORT)

_P = ctypes.c_void_p


class RasterGuard(ctypes.Structure):
    """hs_raster_guard_t"""
    _fields_ = [("summary", ctypes.c_void_p), ("capacity", ctypes.c_uint64), ("longest_max", ctypes.c_uint32)]
_I = ctypes.c_int
_L = ctypes.c_int64
_F = ctypes.c_float
_Z = ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "hs_last_error": (ctypes.c_char_p, []),
    "hs_version": (_I, []),
    "hs_device_sm_count": (_I, [_I]),
    "hs_mlp_size": (_L, [_I, _I, _I]),
    "hs_mlp_fwd": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "hs_mlp_bwd": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "hs_blend_fwd": (_I, [_L, _I, _I, _P, _P, _P, _P, _P]),
    "hs_blend_bwd_kernels": (_I, [_L, _I, _I]),
    "hs_blend_bwd": (_I, [_L, _I, _I, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I), _P]),
    "hs_blend_bwd_partials": (_I, [_L]),
    "hs_project_avatar_fwd": (_I, [_I, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                   _P, _P, _P, _P]),
    "hs_project_world_fwd": (_I, [_I, _L, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hs_project_avatar_bwd": (_I, [_I, _L, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P]),
    "hs_project_world_bwd": (_I, [_I, _L, _P, _P, _P, _P, _P]),
    "hs_scan_blocks": (_I, [_L]),
    "hs_bin_scan": (_I, [_I, _P, _P, _P, _P, _P, _P]),
    "hs_bin_emit": (_I, [_I, _L, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hs_sort_workspace_size": (_Z, [_L]),
    "hs_sort_pairs": (_I, [_L, ctypes.c_uint64, _P, _P, _P, _P, _P, _Z, ctypes.POINTER(_I), _P]),
    "hs_tile_ranges": (_I, [_L, _P, _P, _P]),
    "hs_raster_fwd": (_I, [_I, _L, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hs_raster_bwd": (_I, [_I, _L, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _F, _P, _I, _P, _P]),
    "hs_loss_reduce": (_I, [_I, _I, _I, _I, _P, _P, _P]),
    "hs_raster_train": (_I, [_I, _L, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _F, _P, _P, _P, _P, _P, _P]),
    "hs_raster_workspace_size": (_Z, [_I, _I, _I]),
    "hs_fixed_to_float": (_I, [_L, _P, _P, _I, _P]),
    "hs_depth_order": (_I, [_L, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "hs_bin_emit_sorted": (_I, [_I, _L, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hs_sort_pairs32": (_I, [_L, ctypes.c_uint32, _P, _P, _P, _P, _P, _Z, ctypes.POINTER(_I), _P]),
    "hs_tile_ranges32": (_I, [_L, _P, _P, _P]),
    "hs_tile_sort_cap": (_I, []),
    "hs_tile_cta_sort_min": (_I, []),
    "hs_tile_fill_longest": (_I, [_I, _L, _I, _I, _P, _P, _P, _P, _I, _P, ctypes.c_uint64, _P, _P]),
    "hs_raster_tile_order": (_I, [_I, _I, _I, _P, _I, _P, _P]),
    "hs_tile_count": (_I, [_I, _L, _I, _I, _P, _P, _P, _P]),
    "hs_tile_scan": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "hs_tile_fill": (_I, [_I, _L, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, ctypes.c_uint64, _P, _P, _I, _P, _P]),
    "hs_fork_create": (_P, []),
    "hs_fork_destroy": (None, [_P]),
    "hs_bin_stats": (_I, [ctypes.POINTER(ctypes.c_uint64), _I]),
    "hs_raster_stats": (_I, [ctypes.POINTER(ctypes.c_uint64), _I]),
    "hs_raster_warp_times": (_I, [ctypes.POINTER(ctypes.c_uint64), _I]),
    "hs_adam": (_I, [_L, _I, _L, _P, _P, _P, _P, ctypes.POINTER(_F), _I, _F, _F, _F, _P]),
    "hs_image_metrics": (_I, [_I, _I, _I, _P, _P, _P, _P]),
    "hs_host_register": (_I, [_P, _Z]),
    "hs_host_unregister": (_I, [_P]),
    "hs_gather_rows": (_I, [_I, _L, _P, _P, _P, _P]),
    "hs_rig_frames": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hs_adam_fused": (_I, [_L, _I, _L, _P, _P, _P, _P, ctypes.POINTER(_F), _I, _F, _F, _F, _L, _L, _I, _I, _P, _P,
                           _P, _P, _F, _P, _P, _P, _P]),
    "hs_color_init": (_I, [_I, _L, _P, _P, _F, _P, _P, _P, _P, _P]),
    "hs_color_pack": (_I, [_I, _L, _I, _P, _P, _P, _P]),
    "hs_color_select": (_I, [_I, _L, _I, _P, _P, _P, _P, _P]),
    "hs_color_apply": (_I, [_L, _P, _P, _F, _P, _P, _P, _P]),
    "hs_activate_fwd": (_I, [_L, _P, _P, _P, _P]),
    "hs_activate_bwd": (_I, [_L, _P, _P, _P, _P, _P]),
    "hs_transform_fwd": (_I, [_L, _P, _P, _P, _P, _P, _P]),
    "hs_transform_bwd": (_I, [_L, _P, _P, _P, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()


def header_symbols(path=None):
    """Function names declared in include/hs_api.h."""
    import re
    path = path or os.path.join(os.path.dirname(PKG), "include", "hs_api.h")
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s+\**\s*(hs_[a-z_0-9]+)\s*\(", text, re.M)))


def load():
    """Load the library (raises if absent -- there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2503_12886_b200.build` "
                                   "(the product path has no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().hs_last_error().decode()


def check(rc: int, what: str = ""):
    if rc == HS_OK:
        return
    msg = last_error() or what
    if rc == HS_ERR_SHAPE:
        raise ValueError(msg)
    if rc in (HS_ERR_NONFINITE, HS_ERR_ZERO_QUAT):
        raise FloatingPointError(msg)
    if rc == HS_ERR_COLOR_INIT:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


_FNS = {}


def call(name: str, *args):
    """Call an entry point; raises on a non-zero status (the function objects are
    cached: the per-call cost is on the training step's host path)."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != HS_OK:
        check(rc, name)


ATTR_NAMES = ("position", "rotation", "scale", "opacity", "color")


class DegenerateTriangleError(ValueError):
    """S/binding.py:21-22."""


def raise_device_error(code: int, item_base: int = 0):
    """Map the device error word (hs_api.h) to the reference's exception."""
    if code == HS_NO_ERROR:
        return
    stage = code >> 62
    frame = (code >> 40) & ((1 << 22) - 1)
    attr = (code >> 32) & 0xFF
    n = code & 0xFFFFFFFF
    if stage == 0 and attr == 0:
        raise ValueError("theta contains non-finite values")                      # S/model.py:135-136
    if stage == 0:
        raise FloatingPointError(f"zero-norm quaternion at Gaussian index {n}")    # S/model.py:226-227
    if stage == 1:
        raise FloatingPointError(f"non-finite {ATTR_NAMES[attr]} at Gaussian index {n}")  # S/render.py:208
    if stage == 3:                                                                 # S/binding.py:104-109
        raise DegenerateTriangleError(f"degenerate {'UV' if attr == 0 else '3D'} triangle at face {n}")
    raise RuntimeError(f"Gaussian {n} exceeds the weight threshold but accumulated zero total weight "
                       f"(frame {frame + item_base})")                             # S/color_init.py:59-63
