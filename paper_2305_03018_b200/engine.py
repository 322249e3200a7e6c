"""Plan objects over the C ABI: device tensors in, device tensors out.

A :class:`MorphPlan` owns one ``fm_plan`` (cached SE spectrum, tile geometry,
tonal length, spectral scratch).  It is the batched, device-resident entry
point used by the drop-in operators, the bench and the sharded runner.
torch is used only for device memory and streams.
"""

from __future__ import annotations

import collections
import ctypes
import hashlib
import threading

import numpy as np
import torch

from . import _lib
from ._lib import FM_DILATE, FM_ERODE, FM_I32, FM_U8, FM_U16

# output element types (fm_out_dtype)
_OUT_CODES = {torch.int32: 0, torch.uint8: 1, torch.uint16: 2, torch.int16: 3}


def _torch_dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.uint8:
        return FM_U8
    if t.dtype == torch.uint16:
        return FM_U16
    if t.dtype == torch.int32:
        return FM_I32
    raise TypeError(f"unsupported image dtype {t.dtype} (use uint8, uint16 or int32)")


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class MorphPlan:
    """One precomputed dilation/erosion pipeline for a fixed shape, SE and value range.

    Parameters mirror ``fm_plan_desc`` (include/fftmorph_b200.h).  ``se_values`` /
    ``se_defined`` are host arrays of the SE (``b.values`` / ``b.defined`` of the
    reference's GridFunction) and ``se_lo`` its logical origin ``b.lo``; for
    erosion pass the SE itself — the plan reflects it (morphology.py:147-152).
    """

    def __init__(self, *, shape, se_values, se_lo, se_defined=None, mode="dilate",
                 crop=True, img_dtype=torch.uint8, img_min=0, img_max=255, fill=0,
                 batch=1, device=None, scratch_bytes=0, tile=0, tonal_len=0, out_dtype=torch.int32,
                 counts=False):
        L = _lib.load()
        shape = tuple(int(s) for s in shape)
        se_values = np.ascontiguousarray(np.asarray(se_values, dtype=np.int64))
        if se_values.ndim != len(shape):
            raise ValueError("rank mismatch")
        if np.abs(se_values).max(initial=0) >= 2**31:
            raise NotImplementedError("SE values beyond int32")
        sev = np.ascontiguousarray(se_values.astype(np.int32))
        sed = None if se_defined is None else np.ascontiguousarray(np.asarray(se_defined, dtype=np.uint8))
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", int(device) if not isinstance(device, torch.device) else device.index)
        self.mode = mode
        code = {"dilate": FM_DILATE, "erode": FM_ERODE}[mode]
        d = _lib.PlanDesc()
        d.ndim = len(shape)
        d.mode = code
        d.crop = 1 if crop else 0
        d.img_dtype = {torch.uint8: FM_U8, torch.uint16: FM_U16, torch.int32: FM_I32}[img_dtype]
        d.batch = int(batch)
        for i, s in enumerate(shape):
            d.shape[i] = s
            d.se_shape[i] = int(se_values.shape[i])
            d.se_lo[i] = int(se_lo[i])
        d.img_min = int(img_min)
        d.img_max = int(img_max)
        d.fill = int(fill)
        d.device = self.device.index
        d.scratch_bytes = int(scratch_bytes)
        d.tile = int(tile)
        d.tonal_len = int(tonal_len)
        d.out_dtype = _OUT_CODES[out_dtype]
        d.flags = _lib.FM_FLAG_COUNTS if counts else 0
        self.counts = bool(counts)
        self.out_dtype = out_dtype
        self.desc = d
        self.shape = shape
        self.batch = int(batch)
        self.img_dtype = img_dtype
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            rc = L.fm_plan_create(ctypes.byref(h), ctypes.byref(d),
                                  sev.ctypes.data_as(ctypes.c_void_p),
                                  None if sed is None else sed.ctypes.data_as(ctypes.c_void_p))
        _lib.check(rc)
        self._h = h
        info = _lib.PlanInfo()
        _lib.check(L.fm_plan_query(h, ctypes.byref(info)))
        self.info = {name: (list(getattr(info, name)) if name in ("out_shape", "out_lo_offset")
                            else int(getattr(info, name))) for name, _ in _lib.PlanInfo._fields_}
        nd = len(shape)
        self.out_shape = tuple(self.info["out_shape"][:nd])
        self.out_lo_offset = tuple(self.info["out_lo_offset"][:nd])

    # ------------------------------------------------------------------
    def execute(self, img: torch.Tensor, defined: torch.Tensor | None = None, *,
                out: torch.Tensor | None = None, valid: torch.Tensor | None = None,
                want_valid: bool = True, stream=None):
        """Run on a device batch ``img[batch, *shape]``; returns (out of out_dtype, valid uint8|None)."""
        L = _lib.load()
        if img.device != self.device:
            raise ValueError(f"image on {img.device}, plan on {self.device}")
        if img.dtype != self.img_dtype:
            raise TypeError(f"image dtype {img.dtype} != plan dtype {self.img_dtype}")
        exp = (self.batch, *self.shape)
        if tuple(img.shape) != exp:
            img = img.reshape(exp)
        img = img.contiguous()
        if defined is not None:
            defined = defined.to(device=self.device, dtype=torch.uint8).reshape(exp).contiguous()
        oshape = (self.batch, *self.out_shape)
        if out is None:
            if self.counts:   # count volume [batch, *out_shape, count_len] int32
                out = torch.empty((*oshape, self.info["count_len"]), dtype=torch.int32, device=self.device)
            else:
                out = torch.empty(oshape, dtype=self.out_dtype, device=self.device)
        if valid is None and want_valid:
            valid = torch.empty(oshape, dtype=torch.uint8, device=self.device)
        rc = L.fm_execute(self._h, ctypes.c_void_p(img.data_ptr()),
                          None if defined is None else ctypes.c_void_p(defined.data_ptr()),
                          ctypes.c_void_p(out.data_ptr()),
                          None if valid is None else ctypes.c_void_p(valid.data_ptr()),
                          _stream_ptr(stream))
        _lib.check(rc)
        return out, valid

    def execute_host(self, img: np.ndarray | torch.Tensor, defined=None, *, out=None, valid=None,
                     want_valid=True, stream=None):
        """Host buffers in, host buffers out (copies inside; pinned memory recommended)."""
        L = _lib.load()
        def host(t, dtype):
            if isinstance(t, torch.Tensor):
                assert t.device.type == "cpu" and t.is_contiguous()
                return t
            return torch.from_numpy(np.ascontiguousarray(t)).to(dtype)
        img_t = host(img, self.img_dtype)
        def_t = None if defined is None else host(defined, torch.uint8)
        oshape = (self.batch, *self.out_shape)
        if out is None:
            out = torch.empty(oshape, dtype=self.out_dtype)
        if valid is None and want_valid:
            valid = torch.empty(oshape, dtype=torch.uint8)
        rc = L.fm_execute_host(self._h, ctypes.c_void_p(img_t.data_ptr()),
                               None if def_t is None else ctypes.c_void_p(def_t.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()),
                               None if valid is None else ctypes.c_void_p(valid.data_ptr()),
                               _stream_ptr(stream))
        _lib.check(rc)
        return out, valid

    def set_timing(self, enable: bool) -> None:
        _lib.check(_lib.load().fm_set_timing(self._h, 1 if enable else 0))

    def get_timing(self, reset: bool = False) -> dict:
        t = _lib.Timing()
        _lib.check(_lib.load().fm_get_timing(self._h, ctypes.byref(t), 1 if reset else 0))
        return {name: getattr(t, name) for name, _ in _lib.Timing._fields_}

    def reset_stats(self, stream=None) -> None:
        _lib.check(_lib.load().fm_reset_stats(self._h, _stream_ptr(stream)))

    def read_stats(self, *, raise_errors: bool = True) -> float:
        """Synchronize and return the max pre-rounding deviation since the last reset.

        Raises ArithmeticError if it reached 0.25 (fft_conv.py:145-148) and
        ValueError if an image value fell outside the plan's range."""
        st = _lib.Stats()
        rc = _lib.load().fm_read_stats(self._h, ctypes.byref(st))
        if raise_errors:
            _lib.check(rc)
        return float(st.max_abs_deviation)

    def close(self) -> None:
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.load().fm_plan_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _PlanCache:
    """Small LRU of plans keyed by everything fm_plan_create depends on."""

    def __init__(self, capacity: int = 16):
        self.capacity = capacity
        self._d: collections.OrderedDict = collections.OrderedDict()
        self._mu = threading.Lock()

    def get(self, **kw) -> MorphPlan:
        sev = np.ascontiguousarray(np.asarray(kw["se_values"], dtype=np.int64))
        sed = kw.get("se_defined")
        hsh = hashlib.sha1(sev.tobytes() + (b"" if sed is None else np.asarray(sed, dtype=np.uint8).tobytes()))
        key = (tuple(kw["shape"]), sev.shape, hsh.hexdigest(), tuple(kw["se_lo"]), kw.get("mode", "dilate"),
               bool(kw.get("crop", True)), str(kw.get("img_dtype")), int(kw.get("img_min", 0)),
               int(kw.get("img_max", 255)), int(kw.get("fill", 0)), int(kw.get("batch", 1)),
               str(kw.get("device")), int(kw.get("tile", 0)), int(kw.get("tonal_len", 0)),
               str(kw.get("out_dtype", torch.int32)), int(kw.get("scratch_bytes", 0)))
        with self._mu:
            p = self._d.get(key)
            if p is not None:
                self._d.move_to_end(key)
                return p
        p = MorphPlan(**kw)
        with self._mu:
            self._d[key] = p
            while len(self._d) > self.capacity:
                _, old = self._d.popitem(last=False)
                old.close()
        return p

    def clear(self) -> None:
        with self._mu:
            for p in self._d.values():
                p.close()
            self._d.clear()


plan_cache = _PlanCache()


def naive(*, img: torch.Tensor, defined: torch.Tensor | None, shape, se_values, se_defined, se_lo,
          mode: str, crop: bool, fill: int, batch: int = 1):
    """GPU exact direct operator (fm_naive): dilate_naive / erode_naive semantics."""
    L = _lib.load()
    shape = tuple(int(s) for s in shape)
    sev = np.ascontiguousarray(np.asarray(se_values, dtype=np.int64).astype(np.int32))
    sed = None if se_defined is None else np.ascontiguousarray(np.asarray(se_defined, dtype=np.uint8))
    d = _lib.PlanDesc()
    d.ndim = len(shape)
    d.mode = FM_DILATE if mode == "dilate" else FM_ERODE
    d.crop = 1 if crop else 0
    d.img_dtype = _torch_dtype_code(img)
    d.batch = int(batch)
    for i, s in enumerate(shape):
        d.shape[i] = s
        d.se_shape[i] = int(sev.shape[i])
        d.se_lo[i] = int(se_lo[i])
    d.fill = int(fill)
    d.device = img.device.index
    if crop:
        oshape = shape
    else:
        oshape = tuple(s + m - 1 for s, m in zip(shape, sev.shape))
    out = torch.empty((batch, *oshape), dtype=torch.int32, device=img.device)
    valid = torch.empty((batch, *oshape), dtype=torch.uint8, device=img.device)
    img = img.contiguous()
    if defined is not None:
        defined = defined.to(dtype=torch.uint8).contiguous()
    rc = L.fm_naive(ctypes.byref(d), sev.ctypes.data_as(ctypes.c_void_p),
                    None if sed is None else sed.ctypes.data_as(ctypes.c_void_p),
                    ctypes.c_void_p(img.data_ptr()),
                    None if defined is None else ctypes.c_void_p(defined.data_ptr()),
                    ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(valid.data_ptr()),
                    _stream_ptr(None))
    _lib.check(rc)
    return out, valid
