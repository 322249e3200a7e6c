"""Count-level convolution API on the GPU.

Mirrors ``fftmorph.fft_conv`` (fft_conv.py:46-150): ``next_fast_size``,
``make_plan``, ``direct_full``, ``conv_full_direct``,
``check_precision_budget``, ``conv_full_fft_with_stats`` / ``conv_full_fft``
with the same names, argument meaning, output ranges and errors, so the
reference's count-level tests (test_fft_conv.py:67-139, test_umbra.py:85-123)
read the same against this package.

Operands that are tonal one-hot volumes of 1-D / 2-D grids (``build_umbra``
output: the last axis holds at most one 1 per spatial position) are convolved
by the FFT tile path in count-volume mode (``FM_FLAG_COUNTS``: tonal encode,
spatial FFT convolution, inverse tonal FFT, rounded counts), which is the hot
path of the paper.  Any other non-negative integer operands of rank 1..4
(generic volumes, umbra volumes of 3-D grids, or umbra pairs beyond the tile
path's envelope) go through the FP64 FFT convolution on the device
(``fm_conv_full_fft64``: zero-padded to the reference's ``next_fast_size``
shape, FP64 like the reference, so its 2^52 precision budget applies as is).
``conv_full_direct`` / ``direct_full`` run the exact direct GPU kernel
(``fm_conv_full_direct``).  All arithmetic runs on the device; there is no host
fallback.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import PrecisionBudgetError
from .grid import full_output_range

PRECISION_BUDGET = 2**52          # fft_conv.py:19
MAX_DEVIATION = 0.25              # fft_conv.py:22

_workers = 1


def set_fft_workers(n: int) -> None:
    """API parity with fft_conv.py:27-30 (host FFT threads); the GPU path ignores it."""
    global _workers
    _workers = max(1, int(n))


def get_fft_workers() -> int:
    return _workers


class OffsetArray:
    """Integer array with a logical origin (the role of fftmorph.tensor.OffsetArray)."""

    def __init__(self, data, lo=None):
        self.data = np.asarray(data)
        self.lo = tuple(int(x) for x in (lo if lo is not None else (0,) * self.data.ndim))
        if len(self.lo) != self.data.ndim:
            raise ValueError("lo rank mismatch")

    @property
    def ndim(self):
        return self.data.ndim

    @property
    def shape(self):
        return self.data.shape

    @property
    def hi(self):
        return tuple(l + n - 1 for l, n in zip(self.lo, self.data.shape))

    @property
    def ranges(self):
        return tuple(zip(self.lo, self.hi))

    def at(self, idx):
        rel = tuple(i - l for i, l in zip(idx, self.lo))
        if any(r < 0 or r >= n for r, n in zip(rel, self.data.shape)):
            return 0
        return int(self.data[rel])


@dataclass(frozen=True)
class FftStats:
    """fft_conv.py:54-58."""
    max_abs_deviation: float
    padded_shape: tuple


class Backend(enum.Enum):
    """fft_conv.py:41-43."""
    DIRECT = "direct"
    FFT = "fft"


@dataclass(frozen=True)
class ConvPlan:
    """fft_conv.py:46-51."""
    padded_shape: tuple
    out_lo: tuple
    out_hi: tuple
    backend: Backend


def next_fast_size(n: int) -> int:
    """Smallest of 2^k, 45*2^k that is >= n (fft_conv.py:61-77)."""
    if n < 1:
        raise ValueError("length must be positive")
    pow2 = 1
    while pow2 < n:
        pow2 *= 2
    alt = 45
    while alt < n:
        alt *= 2
    return min(pow2, alt)


def _oa(x):
    if isinstance(x, OffsetArray):
        return x
    if hasattr(x, "data") and hasattr(x, "lo"):       # reference OffsetArray (duck-typed)
        return OffsetArray(x.data, x.lo)
    return OffsetArray(x)


def make_plan(a, b, backend=Backend.FFT) -> ConvPlan:
    """Output range = Minkowski sum; padded = next_fast_size(sa+sb-1) (fft_conv.py:80-91)."""
    a, b = _oa(a), _oa(b)
    if a.ndim != b.ndim:
        raise ValueError("rank mismatch")
    if isinstance(backend, str):
        backend = Backend(backend)
    out_ranges = full_output_range(a.ranges, b.ranges)
    padded = tuple(next_fast_size(sa + sb - 1) for sa, sb in zip(a.shape, b.shape))
    return ConvPlan(padded, tuple(lo for lo, _ in out_ranges), tuple(hi for _, hi in out_ranges), backend)


def check_precision_budget(a, b) -> None:
    """fft_conv.py:114-125: reject min(sum|a| max|b|, sum|b| max|a|) >= 2^52."""
    abs_a = np.abs(np.asarray(a), dtype=np.float64)
    abs_b = np.abs(np.asarray(b), dtype=np.float64)
    bound = min(abs_a.sum() * abs_b.max(), abs_b.sum() * abs_a.max())
    if bound >= PRECISION_BUDGET:
        raise PrecisionBudgetError(f"magnitude bound {bound:.3e} >= 2^52; use the direct backend")


def direct_full(a, b) -> np.ndarray:
    """Full-mode convolution of raw arrays, exact int64, on the GPU (fft_conv.py:94-106)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.int64))
    if a.ndim != b.ndim or not 1 <= a.ndim <= 3:
        raise ValueError("rank mismatch or unsupported rank (1..3)")
    dev = torch.device("cuda", torch.cuda.current_device())
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    out = torch.empty(tuple(sa + sb - 1 for sa, sb in zip(a.shape, b.shape)), dtype=torch.int64, device=dev)
    sa = np.array(a.shape, np.int64)
    sb = np.array(b.shape, np.int64)
    L = _lib.load()
    _lib.check(L.fm_conv_full_direct(a.ndim, sa.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ta.data_ptr()),
                                     sb.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(tb.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()),
                                     ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return out.cpu().numpy()


def conv_full_direct(a, b) -> OffsetArray:
    """fft_conv.py:109-111."""
    plan = make_plan(a, b, Backend.DIRECT)
    a, b = _oa(a), _oa(b)
    return OffsetArray(direct_full(a.data, b.data), plan.out_lo)


def _as_umbra(x: np.ndarray):
    """(values, defined) if x is a tonal one-hot volume of a 1-D / 2-D grid (last axis), else None."""
    if x.ndim < 2 or x.ndim > 3 or x.size == 0:
        return None
    if x.min() < 0 or x.max() > 1:
        return None
    s = x.sum(axis=-1)
    if s.max() > 1:
        return None
    return np.argmax(x, axis=-1).astype(np.int64), s.astype(bool)


def fft64_full(a, b, padded) -> tuple[np.ndarray, float]:
    """Full-mode convolution of two int64 arrays by FP64 FFTs on the device (fm_conv_full_fft64):
    rounded counts and the max pre-rounding deviation (fft_conv.py:133-144)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.int64))
    if a.ndim != b.ndim or not 1 <= a.ndim <= 4:
        raise ValueError("rank mismatch or unsupported rank (1..4)")
    dev = torch.device("cuda", torch.cuda.current_device())
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    out = torch.empty(tuple(sa + sb - 1 for sa, sb in zip(a.shape, b.shape)), dtype=torch.int64, device=dev)
    sa, sb = np.array(a.shape, np.int64), np.array(b.shape, np.int64)
    sp = np.array(padded, np.int64)
    d = ctypes.c_double(0.0)
    L = _lib.load()
    _lib.check(L.fm_conv_full_fft64(a.ndim, sa.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ta.data_ptr()),
                                    sb.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(tb.data_ptr()),
                                    sp.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(out.data_ptr()),
                                    ctypes.byref(d), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    return out.cpu().numpy(), float(d.value)


def _fft64(x: np.ndarray, inverse: bool) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if not 1 <= x.ndim <= 4:
        raise ValueError("unsupported rank (1..4)")
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(x.view(np.float64)).to(dev)
    shp = np.array(x.shape, np.int64)
    _lib.check(_lib.load().fm_fft64(x.ndim, shp.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(t.data_ptr()),
                                    1 if inverse else 0,
                                    ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    out = t.cpu().numpy().view(np.complex128).reshape(x.shape)
    return out / float(np.prod(x.shape)) if inverse else out


def transform_forward(a, plan: ConvPlan) -> np.ndarray:
    """Multidimensional DFT of a real array zero-padded to the plan's shape (fft_conv.py:157-166),
    FP64 on the device."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != len(plan.padded_shape):
        raise ValueError("rank mismatch with plan")
    if any(s > p for s, p in zip(a.shape, plan.padded_shape)):
        raise ValueError("input exceeds the planned transform size")
    z = np.zeros(plan.padded_shape, dtype=np.complex128)
    z[tuple(slice(0, n) for n in a.shape)] = a
    return _fft64(z, inverse=False)


def transform_inverse(spec, plan: ConvPlan) -> np.ndarray:
    """Inverse of transform_forward (fft_conv.py:169-172), FP64 on the device."""
    spec = np.asarray(spec)
    if spec.shape != tuple(plan.padded_shape):
        raise ValueError("spectrum shape does not match plan")
    return _fft64(spec, inverse=True)


def _umbra_counts(fa, fd, fb, bd, out_shape):
    """Count volume of two one-hot volumes through the FFT tile path (FM_FLAG_COUNTS)."""
    from .engine import MorphPlan
    full = np.zeros(out_shape, dtype=np.int64)
    if not fd.any() or not bd.any():
        return full, 0.0
    fv = fa[fd]
    bvals = fb[bd]
    img_min, img_max = int(fv.min()), int(fv.max())
    nd = fa.ndim
    se_lo = (0,) * nd   # counts over the whole Minkowski range; origins handled by the caller
    dt = torch.uint8 if img_max <= 255 else (torch.uint16 if img_max <= 65535 else torch.int32)
    plan = MorphPlan(shape=fa.shape, se_values=fb, se_defined=bd, se_lo=se_lo, mode="dilate", crop=False,
                     img_dtype=dt, img_min=img_min, img_max=img_max, fill=0, counts=True)
    dev = plan.device
    npdt = {torch.uint8: np.uint8, torch.uint16: np.uint16, torch.int32: np.int32}[dt]
    img = torch.from_numpy(np.where(fd, fa, 0).astype(npdt)).to(dev)
    dmask = torch.from_numpy(fd.astype(np.uint8)).to(dev)
    plan.reset_stats()
    counts, _ = plan.execute(img, dmask, want_valid=False)
    dev_max = plan.read_stats()
    c = counts[0].cpu().numpy().astype(np.int64)          # [*spatial_out, l_r + 1]
    base = img_min + int(bvals.min())                     # degree of count index 0
    full[..., base:base + c.shape[-1]] = c[..., :max(0, min(c.shape[-1], out_shape[-1] - base))]
    return full, dev_max


def conv_full_fft_with_stats(a, b):
    """fft_conv.py:128-150: counts over the Minkowski range, rounded, with the deviation check."""
    a, b = _oa(a), _oa(b)
    check_precision_budget(a.data, b.data)
    plan = make_plan(a, b, Backend.FFT)
    out_shape = tuple(h - l + 1 for l, h in zip(plan.out_lo, plan.out_hi))
    ua, ub = _as_umbra(np.asarray(a.data)), _as_umbra(np.asarray(b.data))
    data = None
    if ua is not None and ub is not None:
        # the paper's hot path; convolution commutes, so the operand with the smaller
        # spatial extent takes the SE role (the tile path bounds the SE, not the image)
        (fv, fd), (bv, bd) = (ua, ub) if np.prod(ua[0].shape) >= np.prod(ub[0].shape) else (ub, ua)
        try:
            data, dev = _umbra_counts(fv, fd, bv, bd, out_shape)
        except NotImplementedError:
            data = None       # beyond the tile path's envelope: the FP64 path below
    if data is None:
        data, dev = fft64_full(a.data, b.data, plan.padded_shape)
    if dev >= MAX_DEVIATION:
        raise ArithmeticError(f"pre-rounding deviation {dev:.3g} >= {MAX_DEVIATION}; "
                              "precision budget logic is broken")
    return OffsetArray(data, plan.out_lo), FftStats(max_abs_deviation=float(dev), padded_shape=plan.padded_shape)


def conv_full_fft(a, b) -> OffsetArray:
    """fft_conv.py:153-155."""
    out, _ = conv_full_fft_with_stats(a, b)
    return out
