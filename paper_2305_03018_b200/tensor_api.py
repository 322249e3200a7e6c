"""Batched, device-resident operators on torch tensors (no host round trips).

The drop-in GridFunction API (``morphology.py``) mirrors the reference call
by call; this module is the production entry point for batches already in
HBM, and chains compound operators on the device (SURVEY §8(f) row 1:
``opening`` / ``closing`` / ``beucher_gradient`` of morphology.py:219-239
without leaving the GPU between the erosion and the dilation).

Semantics per call are those of ``dilate_fft`` / ``erode_fft`` with
``crop=True`` on fully defined grids with lo = 0 (optionally a ``defined``
mask): dilation writes 0 where no (image, SE) pair exists, erosion writes
``l`` (default: the image maximum bound), validity is returned as uint8.
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine


def _se_arrays(se, se_defined, se_lo):
    se = np.asarray(se.cpu() if isinstance(se, torch.Tensor) else se, dtype=np.int64)
    sd = None if se_defined is None else np.asarray(
        se_defined.cpu() if isinstance(se_defined, torch.Tensor) else se_defined, dtype=bool)
    if se_lo is None:
        se_lo = tuple(-(s // 2) for s in se.shape)   # centred, as the reference bench (bench.py:94)
    vals = se if sd is None else se[sd]
    if vals.size == 0:
        raise ValueError("grid needs at least one defined pixel")
    return se, sd, tuple(int(x) for x in se_lo), int(vals.min()), int(vals.max())


def _batched(img: torch.Tensor, ndim: int) -> torch.Tensor:
    if not img.is_cuda:
        raise ValueError("tensor_api operators take CUDA tensors (use the GridFunction API for host data)")
    if img.dim() == ndim:
        return img.unsqueeze(0)
    if img.dim() == ndim + 1:
        return img
    raise ValueError(f"expected a [{ndim}]-D image or a batch of them, got shape {tuple(img.shape)}")


def _img_dtype(img: torch.Tensor, lo: int, hi: int):
    if img.dtype in (torch.uint8, torch.uint16, torch.int32):
        return img, img.dtype
    if lo >= 0 and hi <= 255:
        return img.to(torch.uint8), torch.uint8
    if lo >= -(2**31) and hi < 2**31:
        return img.to(torch.int32), torch.int32
    raise NotImplementedError("image values beyond int32")


def _bounds(img: torch.Tensor, defined, img_min, img_max):
    if img_min is None or img_max is None:
        v = img if defined is None else img[defined.bool()]
        if v.numel() == 0:
            raise ValueError("grid needs at least one defined pixel")
        mn, mx = int(v.min().item()), int(v.max().item())
        img_min = mn if img_min is None else img_min
        img_max = mx if img_max is None else img_max
    return int(img_min), int(img_max)


def _run(mode, img, se, se_lo, se_defined, defined, img_min, img_max, fill, out_dtype, *, data_bounds=False):
    se_v, se_d, se_lo, smin, _ = _se_arrays(se, se_defined, se_lo)
    if smin < 0:
        raise ValueError("tonal lift needs non-negative values")
    x = _batched(img, se_v.ndim)
    lo, hi = _bounds(x, defined, img_min, img_max)
    x, dt = _img_dtype(x, lo, hi)
    dmask = None if defined is None else _batched(defined, se_v.ndim)

    def get(pmin, pmax):
        return engine.plan_cache.get(shape=tuple(x.shape[1:]), se_values=se_v, se_defined=se_d, se_lo=se_lo,
                                     mode=mode, crop=True, img_dtype=dt, img_min=pmin, img_max=pmax,
                                     fill=fill, batch=x.shape[0], device=x.device, out_dtype=out_dtype)
    if data_bounds and img_min is None and img_max is None:
        # bounds measured from the data: plan on the normalised range (a cached plan serves
        # every batch of that bit depth; tiles still adapt to the data), exact range fallback
        nmin, nmax = engine.normalized_range(lo, hi)
        if mode == "erode":
            nmax = min(nmax, max(hi, fill))
        nmax = min(nmax, {torch.uint8: 255, torch.uint16: 65535}.get(dt, nmax))
        try:
            plan = get(nmin, nmax)
        except (NotImplementedError, ValueError):
            plan = get(lo, hi)
    else:
        plan = get(lo, hi)
    out, valid = plan.execute(x, dmask)
    if img.dim() == se_v.ndim:
        out, valid = out[0], valid[0]
    return out, valid


def dilate(img, se, se_lo=None, *, se_defined=None, defined=None, img_min=None, img_max=None,
           out_dtype=torch.int32):
    """Exact dilation of a CUDA image or batch; returns (values, validity)."""
    return _run("dilate", img, se, se_lo, se_defined, defined, img_min, img_max, 0, out_dtype,
                data_bounds=True)


def erode(img, se, se_lo=None, *, l=None, se_defined=None, defined=None, img_min=None, img_max=None,
          out_dtype=torch.int32):
    """Exact erosion (erode_fft semantics: ``l`` where no pair exists; default l = image max bound)."""
    x = _batched(img, np.asarray(se.cpu() if isinstance(se, torch.Tensor) else se).ndim)
    lo, hi = _bounds(x, defined, img_min, img_max)
    if l is None:
        l = hi
    if l < hi:
        raise ValueError(f"l={l} below max value {hi}")
    if img_min is None and img_max is None:
        return _run("erode", img, se, se_lo, se_defined, defined, None, None, int(l), out_dtype, data_bounds=True)
    return _run("erode", img, se, se_lo, se_defined, defined, lo, hi, int(l), out_dtype)


def _range_after_erosion(lo, hi, se_min, se_max, l):
    return min(lo - se_max, l), max(hi - se_min, l)


def opening(img, se, se_lo=None, *, l=None, se_defined=None):
    """dilate(erode(f)) on the device (morphology.py:219-222)."""
    se_v, se_d, lo_se, smin, smax = _se_arrays(se, se_defined, se_lo)
    x = _batched(img, se_v.ndim)
    lo, hi = _bounds(x, None, None, None)
    l = hi if l is None else int(l)
    e, _ = erode(img, se_v, lo_se, l=l, se_defined=se_d, img_min=lo, img_max=hi)
    elo, ehi = _range_after_erosion(lo, hi, smin, smax, l)
    d, _ = dilate(e, se_v, lo_se, se_defined=se_d, img_min=elo, img_max=ehi)
    return d


def closing(img, se, se_lo=None, *, l=None, se_defined=None):
    """erode(dilate(f), l = dilation tonal ceiling) on the device (morphology.py:225-229).

    With no explicit ``l`` the ceiling is max f + max b (the dilation's
    tonal_max for an image whose declared ceiling is its maximum)."""
    se_v, se_d, lo_se, smin, smax = _se_arrays(se, se_defined, se_lo)
    x = _batched(img, se_v.ndim)
    lo, hi = _bounds(x, None, None, None)
    d, _ = dilate(img, se_v, lo_se, se_defined=se_d, img_min=lo, img_max=hi)
    dlo, dhi = min(lo + smin, 0), hi + smax
    l = max(hi + smax, 1) if l is None else int(l)
    e, _ = erode(d, se_v, lo_se, l=l, se_defined=se_d, img_min=dlo, img_max=dhi)
    return e


def gradient(img, se, se_lo=None, *, l=None, se_defined=None):
    """Beucher gradient max(dilate - erode, 0) on the device (morphology.py:232-239)."""
    se_v, se_d, lo_se, _, _ = _se_arrays(se, se_defined, se_lo)
    x = _batched(img, se_v.ndim)
    lo, hi = _bounds(x, None, None, None)
    d, _ = dilate(img, se_v, lo_se, se_defined=se_d, img_min=lo, img_max=hi)
    e, _ = erode(img, se_v, lo_se, l=hi if l is None else int(l), se_defined=se_d, img_min=lo, img_max=hi)
    return torch.clamp(d - e, min=0)
