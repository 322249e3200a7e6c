"""Count-level types and maps of the paper's pipeline, device-backed.

Same names, fields and semantics as ``fftmorph.umbra`` (umbra.py:135-210):
``UmbraVolume`` / ``CountVolume`` (with ``verify``), ``required_lr``,
``build_umbra``, ``project`` and ``project_with_validity``, so the reference's
count-level tests (test_umbra.py, test_fft_conv.py) read the same against this
package.  The volume-building and projection arithmetic runs in the sm_100a
library (``fm_build_umbra`` / ``fm_project``, csrc/fm_fft64.cuh); this module
does the host bookkeeping the reference does (validation, ``lo`` arithmetic,
range checks).  Volumes are returned as host ``OffsetArray``s like the
reference's (its tests slice ``.data`` with numpy).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .fft_conv import OffsetArray
from .grid import GridFunction, intersect_ranges


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2305_03018_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


@dataclass(frozen=True)
class UmbraVolume:
    """(N+1)-d 0/1 volume: spatial axes of the source grid x tonal axis [0..l_R] (umbra.py:135-152)."""
    bits: OffsetArray
    l_R: int

    @property
    def spatial_ranges(self):
        return self.bits.ranges[:-1]

    def verify(self) -> None:
        data = self.bits.data
        if not np.isin(data, (0, 1)).all():
            raise AssertionError("umbra entries must be 0/1")
        if (data.sum(axis=-1) > 1).any():
            raise AssertionError("more than one 1 in a tonal column")


@dataclass(frozen=True)
class CountVolume:
    """(N+1)-d non-negative counts: full-conv output of two umbra volumes (umbra.py:154-169)."""
    counts: OffsetArray
    l_R: int

    @property
    def spatial_ranges(self):
        return self.counts.ranges[:-1]

    def verify(self) -> None:
        data = self.counts.data
        if data.min() < 0:
            raise AssertionError("negative count")
        if data.shape[-1] > self.l_R + 1 and data[..., self.l_R + 1:].any():
            raise AssertionError("nonzero count above the achievable degree")


def required_lr(f, b) -> int:
    """Shared tonal extent of the two lifted volumes: max f + max b (umbra.py:172-174)."""
    f, b = GridFunction.coerce(f), GridFunction.coerce(b)
    return f.max_defined() + b.max_defined()


def build_umbra(g, l_R: int) -> UmbraVolume:
    """Tonal lift (umbra.py:177-186) on the device: bits[x, g(x)] = 1 at defined x."""
    g = GridFunction.coerce(g)
    l_R = int(l_R)
    if l_R < g.max_defined():
        raise ValueError(f"l_R={l_R} below max value {g.max_defined()}")
    if g.min_defined() < 0:
        raise ValueError("cannot lift negative values")
    dev = _dev()
    t = l_R + 1
    vals = torch.from_numpy(np.array(g.values, dtype=np.int64, copy=True)).to(dev)
    mask = None if g.gap_free else torch.from_numpy(g.defined.astype(np.uint8)).to(dev)
    bits = torch.empty((*g.shape, t), dtype=torch.int64, device=dev)
    _lib.check(_lib.load().fm_build_umbra(int(np.prod(g.shape)), ctypes.c_void_p(vals.data_ptr()),
                                          None if mask is None else ctypes.c_void_p(mask.data_ptr()),
                                          t, ctypes.c_void_p(bits.data_ptr()), _stream(dev)))
    return UmbraVolume(OffsetArray(bits.cpu().numpy(), tuple(g.lo) + (0,)), l_R)


def project_with_validity(c: CountVolume, out_range) -> tuple[GridFunction, np.ndarray]:
    """Top tonal index with count >= 1 per pixel of ``out_range`` and the mask of non-empty
    columns (umbra.py:189-205), reduced on the device."""
    counts = c.counts if isinstance(c.counts, OffsetArray) else OffsetArray(c.counts.data, c.counts.lo)
    spatial = counts.ranges[:-1]
    out_range = tuple(tuple(int(v) for v in r) for r in out_range)
    if intersect_ranges(spatial, out_range) != out_range:
        raise ValueError(f"out_range {out_range} outside volume {spatial}")
    sl = tuple(slice(lo - clo, hi - clo + 1) for (lo, hi), (clo, _) in zip(out_range, spatial))
    window = np.ascontiguousarray(np.asarray(counts.data)[sl], dtype=np.int64)
    shape = window.shape[:-1]
    t = window.shape[-1]
    npx = int(np.prod(shape))
    dev = _dev()
    w = torch.from_numpy(window).to(dev)
    values = torch.empty(shape, dtype=torch.int64, device=dev)
    valid = torch.empty(shape, dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().fm_project(npx, t, ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(values.data_ptr()),
                                      ctypes.c_void_p(valid.data_ptr()), _stream(dev)))
    v = values.cpu().numpy()
    g = GridFunction(v, lo=tuple(lo for lo, _ in out_range),
                     tonal_max=max(int(c.l_R), int(v.max(initial=0)), 1))
    return g, valid.cpu().numpy().astype(bool)


def project(c: CountVolume, out_range) -> GridFunction:
    """Top nonzero tonal index per spatial pixel; 0 where the column is empty (umbra.py:208-210)."""
    return project_with_validity(c, out_range)[0]
