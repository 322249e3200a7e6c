"""ORACLE — test infrastructure only.  ctypes wrapper of oracle/naive.c.

Exact dilate_naive / erode_naive (morphology.py:65-113) in C, multithreaded,
for checking the GPU path at full BASELINE sizes.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_LIB = _DIR / "_build" / "libmorph_oracle.so"
_lib = None


def build() -> Path:
    src = _DIR / "naive.c"
    if not _LIB.exists() or _LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        vp = ctypes.c_void_p
        L.oracle_naive.argtypes = [ctypes.c_int, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int32, vp, vp, ctypes.c_int]
        L.oracle_naive.restype = ctypes.c_int
        _lib = L
    return _lib


def naive(img, img_def, se, se_def, se_lo, *, erode=False, crop=True, fill=0, threads=None):
    """Returns (values int32, valid bool) for one 1-D or 2-D image (image lo = 0)."""
    L = _load()
    img = np.ascontiguousarray(np.asarray(img).astype(np.int32))
    se = np.ascontiguousarray(np.asarray(se).astype(np.int32))
    ndim = img.ndim
    shape = np.array(img.shape, np.int64)
    sshape = np.array(se.shape, np.int64)
    slo = np.array(se_lo, np.int64)
    idf = None if img_def is None else np.ascontiguousarray(np.asarray(img_def, np.uint8))
    sdf = None if se_def is None else np.ascontiguousarray(np.asarray(se_def, np.uint8))
    if crop:
        oshape = img.shape
    else:
        oshape = tuple(s + m - 1 for s, m in zip(img.shape, se.shape))
    out = np.empty(oshape, np.int32)
    valid = np.empty(oshape, np.uint8)
    p = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)
    rc = L.oracle_naive(ndim, p(shape), p(img), p(idf), p(sshape), p(se), p(sdf), p(slo),
                        1 if erode else 0, 1 if crop else 0, int(fill), p(out), p(valid),
                        threads or len(os.sched_getaffinity(0)))
    if rc:
        raise RuntimeError("oracle_naive failed")
    return out, valid.astype(bool)
