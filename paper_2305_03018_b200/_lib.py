"""ctypes binding of the C ABI in include/fftmorph_b200.h.

This is the exact binding a maintainer of the reference would add next to
``fftmorph.morphology``.  The library is built in-tree by
``paper_2305_03018_b200.build`` / ``__graft_entry__.build()``; if it is absent
every operator raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_build" / "libfftmorph_b200.so"
if os.environ.get("FM_LIB"):   # A/B builds for measurements (must still be an in-tree build)
    LIB_PATH = Path(os.environ["FM_LIB"]).resolve()

ABI_VERSION = 4   # FM_ABI_VERSION of include/fftmorph_b200.h
FM_OK, FM_EINVAL, FM_EPRECISION, FM_EDEVIATION, FM_ECUDA, FM_EUNSUPPORTED, FM_ENOMEM = range(7)
FM_DILATE, FM_ERODE = 0, 1
FM_U8, FM_U16, FM_I32 = 0, 1, 2
FM_OUT_I32, FM_OUT_U8, FM_OUT_U16, FM_OUT_I16 = 0, 1, 2, 3

# every symbol the header declares (checked by the CPU test-suite)
EXPORTED = (
    "fm_plan_create", "fm_execute", "fm_execute_host", "fm_read_stats", "fm_reset_stats",
    "fm_plan_query", "fm_plan_destroy", "fm_naive", "fm_kernel_launches", "fm_last_error",
    "fm_abi_version", "fm_set_timing", "fm_get_timing", "fm_conv_full_direct",
    "fm_conv_full_fft64", "fm_fft64", "fm_build_umbra", "fm_project",
    "fm_copy_peer", "fm_ipc_get_handle", "fm_ipc_open_handle", "fm_ipc_close_handle",
)
FM_FLAG_COUNTS = 1


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("crop", ctypes.c_int32),
        ("img_dtype", ctypes.c_int32),
        ("batch", ctypes.c_int64),
        ("shape", ctypes.c_int64 * 2),
        ("se_shape", ctypes.c_int64 * 2),
        ("se_lo", ctypes.c_int64 * 2),
        ("img_min", ctypes.c_int32),
        ("img_max", ctypes.c_int32),
        ("fill", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("scratch_bytes", ctypes.c_int64),
        ("tile", ctypes.c_int32),
        ("tonal_len", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("count_budget", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("win_lo", ctypes.c_int64 * 2),
        ("win_shape", ctypes.c_int64 * 2),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("tonal_len", ctypes.c_int32),
        ("planes", ctypes.c_int32),
        ("l_r", ctypes.c_int32),
        ("tile_y", ctypes.c_int32),
        ("tile_x", ctypes.c_int32),
        ("valid_y", ctypes.c_int32),
        ("valid_x", ctypes.c_int32),
        ("tiles_y", ctypes.c_int32),
        ("tiles_x", ctypes.c_int32),
        ("k_chunk", ctypes.c_int32),
        ("out_shape", ctypes.c_int64 * 2),
        ("out_lo_offset", ctypes.c_int64 * 2),
        ("images_per_launch", ctypes.c_int64),
        ("scratch_bytes", ctypes.c_int64),
        ("se_min", ctypes.c_int32),
        ("se_max", ctypes.c_int32),
        ("se_count", ctypes.c_int32),
        ("count_len", ctypes.c_int32),
    ]


class Timing(ctypes.Structure):
    _fields_ = [("conv_ms", ctypes.c_double), ("tonal_ms", ctypes.c_double),
                ("conv_launches", ctypes.c_int64), ("tonal_launches", ctypes.c_int64),
                ("conv_bytes", ctypes.c_double), ("tonal_bytes", ctypes.c_double),
                ("conv_flops", ctypes.c_double), ("range_ms", ctypes.c_double),
                ("range_launches", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("max_abs_deviation", ctypes.c_double), ("value_error", ctypes.c_int32)]


_lock = threading.Lock()
_lib = None


def lib_available() -> bool:
    return LIB_PATH.exists()


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is not built; run `python -m paper_2305_03018_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.fm_plan_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(PlanDesc), vp, vp]
        L.fm_plan_create.restype = ctypes.c_int
        L.fm_execute.argtypes = [vp, vp, vp, vp, vp, vp]
        L.fm_execute.restype = ctypes.c_int
        L.fm_execute_host.argtypes = [vp, vp, vp, vp, vp, vp]
        L.fm_execute_host.restype = ctypes.c_int
        L.fm_read_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.fm_read_stats.restype = ctypes.c_int
        L.fm_reset_stats.argtypes = [vp, vp]
        L.fm_reset_stats.restype = ctypes.c_int
        L.fm_plan_query.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.fm_plan_query.restype = ctypes.c_int
        L.fm_plan_destroy.argtypes = [vp]
        L.fm_plan_destroy.restype = None
        L.fm_naive.argtypes = [ctypes.POINTER(PlanDesc), vp, vp, vp, vp, vp, vp, vp]
        L.fm_naive.restype = ctypes.c_int
        L.fm_kernel_launches.argtypes = []
        L.fm_kernel_launches.restype = i64
        L.fm_last_error.argtypes = []
        L.fm_last_error.restype = ctypes.c_char_p
        L.fm_set_timing.argtypes = [vp, ctypes.c_int]
        L.fm_set_timing.restype = ctypes.c_int
        L.fm_get_timing.argtypes = [vp, ctypes.POINTER(Timing), ctypes.c_int]
        L.fm_get_timing.restype = ctypes.c_int
        L.fm_abi_version.argtypes = []
        L.fm_abi_version.restype = i32
        L.fm_conv_full_direct.argtypes = [ctypes.c_int, vp, vp, vp, vp, vp, vp]
        L.fm_conv_full_direct.restype = ctypes.c_int
        L.fm_conv_full_fft64.argtypes = [ctypes.c_int, vp, vp, vp, vp, vp, vp, ctypes.POINTER(ctypes.c_double), vp]
        L.fm_conv_full_fft64.restype = ctypes.c_int
        L.fm_fft64.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, vp]
        L.fm_fft64.restype = ctypes.c_int
        L.fm_build_umbra.argtypes = [i64, vp, vp, i64, vp, vp]
        L.fm_build_umbra.restype = ctypes.c_int
        L.fm_project.argtypes = [i64, i64, vp, vp, vp, vp]
        L.fm_project.restype = ctypes.c_int
        L.fm_copy_peer.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, i64, vp]
        L.fm_copy_peer.restype = ctypes.c_int
        L.fm_ipc_get_handle.argtypes = [vp, vp, ctypes.POINTER(i64)]
        L.fm_ipc_get_handle.restype = ctypes.c_int
        L.fm_ipc_open_handle.argtypes = [vp, ctypes.c_int, ctypes.POINTER(vp)]
        L.fm_ipc_open_handle.restype = ctypes.c_int
        L.fm_ipc_close_handle.argtypes = [vp]
        L.fm_ipc_close_handle.restype = ctypes.c_int
        _lib = L
        return L


class PrecisionBudgetError(ValueError):
    """Same role as fftmorph.fft_conv.PrecisionBudgetError (fft_conv.py:37-38)."""


def check(rc: int) -> None:
    """Map an fm_status to the reference's exception types."""
    if rc == FM_OK:
        return
    msg = load().fm_last_error().decode(errors="replace")
    if rc == FM_EINVAL:
        raise ValueError(msg)
    if rc == FM_EPRECISION:
        raise PrecisionBudgetError(msg)
    if rc == FM_EDEVIATION:
        raise ArithmeticError(msg)
    if rc == FM_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == FM_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def kernel_launches() -> int:
    return int(load().fm_kernel_launches())
