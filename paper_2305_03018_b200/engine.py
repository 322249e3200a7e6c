"""Plan objects over the C ABI: device tensors in, device tensors out.

A :class:`MorphPlan` owns one ``fm_plan`` (cached SE spectrum, tile geometry,
tonal length, spectral scratch).  It is the batched, device-resident entry
point used by the drop-in operators, the bench and the sharded runner.
torch is used only for device memory and streams.
"""

from __future__ import annotations

import collections
import ctypes
import math
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


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(stream, device_index: int | None = None) -> ctypes.c_void_p:
    """CUDA stream handle of `stream` (default: torch's current stream of the device).  The raw
    query is ~50x cheaper than building a torch.cuda.Stream object, which matters for small calls."""
    if stream is None:
        if _raw_stream is not None:
            if device_index is None:
                device_index = torch.cuda.current_device()
            return ctypes.c_void_p(_raw_stream(device_index))
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
                 counts=False, count_budget=0, window=None):
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
        if window is not None:
            # explicit output window (row strips): ((lo per axis), (shape per axis)) in
            # image-array indices; crop is ignored
            wlo, wsh = window
            if len(wlo) != len(shape) or len(wsh) != len(shape):
                raise ValueError("window rank mismatch")
            d.crop = 2
            for i in range(len(shape)):
                d.win_lo[i] = int(wlo[i])
                d.win_shape[i] = int(wsh[i])
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
        d.count_budget = int(count_budget)
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
    # ------------------------------------------------------------------
    def _check(self, t, name, shape, dtype, device, *, numel_only=False):
        """Raise (ValueError / TypeError) unless `t` is a contiguous tensor of `shape` and `dtype`
        on `device`: raw pointers go to the library, so a wrong buffer must never reach it."""
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
        if t.dtype != dtype:
            raise TypeError(f"{name} dtype {t.dtype} != expected {dtype}")
        if t.device != device:
            raise ValueError(f"{name} on {t.device}, expected {device}")
        n = math.prod(int(x) for x in shape)
        if t.numel() != n or (not numel_only and tuple(t.shape) != tuple(shape)):
            raise ValueError(f"{name} shape {tuple(t.shape)} != expected {tuple(shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")

    def _out_shapes(self):
        oshape = (self.batch, *self.out_shape)
        vshape = oshape
        if self.counts:   # count volume [batch, *out_shape, count_len] int32
            oshape = (*oshape, self.info["count_len"])
        return oshape, vshape, (torch.int32 if self.counts else self.out_dtype)

    def execute(self, img: torch.Tensor, defined: torch.Tensor | None = None, *,
                out: torch.Tensor | None = None, valid: torch.Tensor | None = None,
                want_valid: bool = True, stream=None):
        """Run on a device batch ``img[batch, *shape]``; returns (out of out_dtype, valid uint8|None)."""
        L = _lib.load()
        exp = (self.batch, *self.shape)
        if not isinstance(img, torch.Tensor):
            raise TypeError("img must be a torch.Tensor on the plan's device")
        if img.device != self.device:
            raise ValueError(f"image on {img.device}, plan on {self.device}")
        if img.dtype != self.img_dtype:
            raise TypeError(f"image dtype {img.dtype} != plan dtype {self.img_dtype}")
        if img.numel() != math.prod(exp):
            raise ValueError(f"image shape {tuple(img.shape)} does not hold a batch of {exp}")
        img = img.reshape(exp).contiguous()
        if defined is not None:
            if not isinstance(defined, torch.Tensor) or defined.numel() != img.numel():
                raise ValueError("defined mask must be a tensor with the image's element count")
            defined = defined.to(device=self.device, dtype=torch.uint8).reshape(exp).contiguous()
        oshape, vshape, odt = self._out_shapes()
        if out is None:
            out = torch.empty(oshape, dtype=odt, device=self.device)
        else:
            self._check(out, "out", oshape, odt, self.device)
        if valid is None and want_valid:
            valid = torch.empty(vshape, dtype=torch.uint8, device=self.device)
        elif valid is not None:
            self._check(valid, "valid", vshape, torch.uint8, self.device)
        rc = L.fm_execute(self._h, ctypes.c_void_p(img.data_ptr()),
                          None if defined is None else ctypes.c_void_p(defined.data_ptr()),
                          ctypes.c_void_p(out.data_ptr()),
                          None if valid is None else ctypes.c_void_p(valid.data_ptr()),
                          _stream_ptr(stream, self.device.index))
        _lib.check(rc)
        return out, valid

    def execute_host(self, img: np.ndarray | torch.Tensor, defined=None, *, out=None, valid=None,
                     want_valid=True, stream=None):
        """Host buffers in, host buffers out (copies inside; pinned memory recommended)."""
        L = _lib.load()
        if self.counts:
            raise NotImplementedError("count-volume plans run on device buffers (execute)")
        cpu = torch.device("cpu")
        exp = (self.batch, *self.shape)

        def host(t, dtype, name):
            if isinstance(t, torch.Tensor):
                self._check(t, name, exp, dtype, cpu, numel_only=True)
                return t
            a = np.ascontiguousarray(t)
            if a.size != math.prod(exp):
                raise ValueError(f"{name} shape {a.shape} does not hold a batch of {exp}")
            return torch.from_numpy(a).to(dtype)
        img_t = host(img, self.img_dtype, "img")
        def_t = None if defined is None else host(defined, torch.uint8, "defined")
        oshape = (self.batch, *self.out_shape)
        if out is None:
            out = torch.empty(oshape, dtype=self.out_dtype)
        else:
            self._check(out, "out", oshape, self.out_dtype, cpu)
        if valid is None and want_valid:
            valid = torch.empty(oshape, dtype=torch.uint8)
        elif valid is not None:
            self._check(valid, "valid", oshape, torch.uint8, cpu)
        rc = L.fm_execute_host(self._h, ctypes.c_void_p(img_t.data_ptr()),
                               None if def_t is None else ctypes.c_void_p(def_t.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()),
                               None if valid is None else ctypes.c_void_p(valid.data_ptr()),
                               _stream_ptr(stream, self.device.index))
        _lib.check(rc)
        return out, valid

    def set_timing(self, enable: bool) -> None:
        _lib.check(_lib.load().fm_set_timing(self._h, 1 if enable else 0))

    def get_timing(self, reset: bool = False) -> dict:
        t = _lib.Timing()
        _lib.check(_lib.load().fm_get_timing(self._h, ctypes.byref(t), 1 if reset else 0))
        return {name: getattr(t, name) for name, _ in _lib.Timing._fields_}

    def reset_stats(self, stream=None) -> None:
        _lib.check(_lib.load().fm_reset_stats(self._h, _stream_ptr(stream, self.device.index)))

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


def normalized_range(vmin: int, vmax: int) -> tuple[int, int]:
    """Plan key for a data range: the smallest [0, 2^k - 1] holding it (non-negative data), else
    [-(2^k), 2^k - 1].  Plans are built for the normalised range -- exact for every value inside
    it (the per-tile range kernel still adapts each tile's tonal length to the data) -- so a new
    image with a slightly different min/max reuses the cached plan instead of building one."""
    vmin, vmax = int(vmin), int(vmax)
    if vmin >= 0:
        top = 1
        while top < vmax:
            top = 2 * top + 1
        return 0, top
    m = 1
    while -m > vmin or m - 1 < vmax:
        m *= 2
    return -m, m - 1


class _PlanCache:
    """LRU of plans keyed by everything fm_plan_create depends on, bounded by the device scratch
    the cached plans hold (default 24 GiB, FM_PLAN_CACHE_GIB), not by their count.  A plan whose
    creation runs out of device memory evicts every cached plan and is retried once."""

    def __init__(self, capacity: int = 32, max_bytes: int | None = None):
        import os
        self.capacity = capacity
        self.max_bytes = max_bytes if max_bytes is not None else int(
            float(os.environ.get("FM_PLAN_CACHE_GIB", "24")) * (1 << 30))
        self._d: collections.OrderedDict = collections.OrderedDict()
        self._mu = threading.Lock()

    @staticmethod
    def _bytes(p: MorphPlan) -> int:
        return int(p.info.get("scratch_bytes", 0))

    def held_bytes(self) -> int:
        with self._mu:
            return sum(self._bytes(p) for p in self._d.values())

    def _evict_locked(self, need: int = 0):
        while self._d and (len(self._d) >= self.capacity or
                           sum(self._bytes(p) for p in self._d.values()) + need > self.max_bytes):
            _, old = self._d.popitem(last=False)
            old.close()

    def get(self, **kw) -> MorphPlan:
        sev = np.ascontiguousarray(np.asarray(kw["se_values"], dtype=np.int64))
        sed = kw.get("se_defined")
        hsh = hashlib.sha1(sev.tobytes() + (b"" if sed is None else np.asarray(sed, dtype=np.uint8).tobytes()))
        key = (tuple(kw["shape"]), sev.shape, hsh.hexdigest(), tuple(kw["se_lo"]), kw.get("mode", "dilate"),
               bool(kw.get("crop", True)), str(kw.get("img_dtype")), int(kw.get("img_min", 0)),
               int(kw.get("img_max", 255)), int(kw.get("fill", 0)), int(kw.get("batch", 1)),
               str(kw.get("device")), int(kw.get("tile", 0)), int(kw.get("tonal_len", 0)),
               str(kw.get("out_dtype", torch.int32)), int(kw.get("scratch_bytes", 0)),
               bool(kw.get("counts", False)), int(kw.get("count_budget", 0)), repr(kw.get("window")))
        with self._mu:
            p = self._d.get(key)
            if p is not None:
                self._d.move_to_end(key)
                return p
        try:
            p = MorphPlan(**kw)
        except MemoryError:
            self.clear()
            torch.cuda.empty_cache()
            p = MorphPlan(**kw)
        with self._mu:
            self._evict_locked(self._bytes(p))
            self._d[key] = p
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
