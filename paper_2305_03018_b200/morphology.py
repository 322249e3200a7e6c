"""Drop-in operators: the reference's dilation / erosion entry points on B200.

Same names, signatures, argument meaning, return types and error behaviour as
``fftmorph.morphology`` (reference morphology.py:30-239).  The value
computation of every FFT operator runs in the sm_100a library through
:class:`~paper_2305_03018_b200.engine.MorphPlan`; this module does only the
host bookkeeping the reference does in Python (validation, ``lo`` / range
arithmetic, ``tonal_max``, ``stats``).  The ``naive`` method runs the GPU
direct kernel (same semantics as dilate_naive / erode_naive); nothing here
computes image values on the CPU.
"""

from __future__ import annotations

import enum
import warnings

import numpy as np
import torch

from . import engine
from .grid import GridFunction, full_output_range, intersect_ranges


class MorphMethod(enum.Enum):
    """morphology.py:30-41."""
    NAIVE = "naive"
    FFT_UMBRA = "fft"

    @classmethod
    def parse(cls, name) -> "MorphMethod":
        if isinstance(name, cls):
            return name
        for m in cls:
            if name in (m.value, m.name, m.name.lower()):
                return m
        raise ValueError(f"unknown method {name!r}")


# --------------------------------------------------------------------------- helpers

_cuda_ok = False


def _device():
    global _cuda_ok
    if not _cuda_ok:   # (checked once: the query costs ~7 us per call)
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2305_03018_b200 needs a CUDA device (B200); there is no CPU fallback")
        _cuda_ok = True
    return torch.device("cuda", torch.cuda.current_device())


def _upload(g: GridFunction, dev):
    """Device copy of a grid's values in the narrowest supported dtype, plus its mask."""
    vals = g.values
    lo_v, hi_v = g.min_defined(), g.max_defined()
    if lo_v >= 0 and hi_v <= 255:
        dt, npdt = torch.uint8, np.uint8
    elif lo_v >= 0 and hi_v <= 65535:
        dt, npdt = torch.uint16, np.uint16
    elif lo_v >= -(2**31) and hi_v < 2**31:
        dt, npdt = torch.int32, np.int32
    else:
        raise NotImplementedError("image values beyond int32")
    # narrowing int64 -> the device type with torch's multithreaded CPU kernels (numpy's
    # astype is single-threaded: ~3 ms for a 2048^2 image), staged in pinned memory
    with warnings.catch_warnings():   # the grid's arrays are read-only by contract; only read here
        warnings.simplefilter("ignore", UserWarning)
        src = torch.from_numpy(np.ascontiguousarray(vals))
        if not g.gap_free:
            src = torch.where(torch.from_numpy(np.ascontiguousarray(g.defined)), src, torch.zeros((), dtype=src.dtype))
    host = torch.empty(src.shape, dtype=dt, pin_memory=True)
    host.copy_(src)
    t = host.to(dev, non_blocking=True)
    mask = None if g.gap_free else torch.from_numpy(g.defined.astype(np.uint8)).to(dev)
    return t, mask, dt, lo_v, hi_v


import os as _os

# grids up to this size take the one-call host-buffer path (FM_SMALL_ELEMS overrides, for measurements)
_SMALL_ELEMS = int(_os.environ.get("FM_SMALL_ELEMS", 1 << 16))


def _narrow_dtype(g: GridFunction):
    lo_v, hi_v = g.min_defined(), g.max_defined()
    if lo_v >= 0 and hi_v <= 255:
        return torch.uint8, lo_v, hi_v
    if lo_v >= 0 and hi_v <= 65535:
        return torch.uint16, lo_v, hi_v
    if lo_v >= -(2**31) and hi_v < 2**31:
        return torch.int32, lo_v, hi_v
    raise NotImplementedError("image values beyond int32")


def _run_fft(f: GridFunction, b: GridFunction, *, mode: str, crop: bool, fill: int,
             stats: dict | None):
    dev = _device()
    small = f.values.size <= _SMALL_ELEMS
    if small:
        # small grids: the call is bound by its fixed costs, so it is ONE library call on host
        # buffers (fm_execute_host: upload, kernels, download, synchronise) instead of pinned
        # staging tensors, device tensors, an extrema kernel and four stream operations
        dt, vmin, vmax = _narrow_dtype(f)
        img = mask = None
    else:
        img, mask, dt, vmin, vmax = _upload(f, dev)
    # plans are keyed on the normalised range [0, 2^k - 1] holding the data (the per-tile
    # range kernel adapts every tile's tonal length to the data itself), so images of one
    # bit depth share a cached plan; the exact range is the fallback when the wider one
    # exceeds a tonal-length limit
    def get(pmin, pmax):
        # narrowest output element type holding every possible result (fewer bytes
        # back over the bus; widened to int64 on the host like the reference's)
        bmin, bmax = b.min_defined(), b.max_defined()
        if mode == "dilate":
            olo, ohi = min(fill, pmin + bmin), max(fill, pmax + bmax)
        else:
            olo, ohi = min(fill, pmin - bmax), max(fill, pmax - bmin)
        if 0 <= olo and ohi <= 255:
            odt = torch.uint8
        elif -32768 <= olo and ohi <= 32767:
            odt = torch.int16
        else:
            odt = torch.int32
        return engine.plan_cache.get(
            shape=f.shape, se_values=b.values, se_defined=None if b.gap_free else b.defined,
            se_lo=b.lo, mode=mode, crop=crop, img_dtype=dt, img_min=pmin, img_max=pmax,
            fill=fill, batch=1, device=dev, out_dtype=odt)
    nmin, nmax = engine.normalized_range(vmin, vmax)
    if mode == "erode":
        # erode_fft passes l as the fill; the erosion encode uses the plan's max (exact for
        # any bound >= the data max), kept <= l so the fill stays the largest output
        nmax = min(nmax, max(vmax, fill))
    if dt == torch.uint8:
        nmax = min(nmax, 255)
    elif dt == torch.uint16:
        nmax = min(nmax, 65535)
    try:
        plan = get(nmin, nmax)
    except NotImplementedError:
        if (nmin, nmax) == (vmin, vmax):
            raise
        plan = get(vmin, vmax)
    plan.reset_stats()
    if small:
        with warnings.catch_warnings():   # read-only arrays by contract; only read here
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(np.ascontiguousarray(f.values))
            if f.gap_free:
                h_mask = None
            else:
                h_def = torch.from_numpy(np.ascontiguousarray(f.defined))
                src = torch.where(h_def, src, torch.zeros((), dtype=src.dtype))
                h_mask = h_def.to(torch.uint8)
        out, valid = plan.execute_host(src.to(dt), h_mask)
    else:
        out, valid = plan.execute(img.unsqueeze(0), None if mask is None else mask.unsqueeze(0))
    dev_max = plan.read_stats()          # raises ArithmeticError at >= 0.25 (fft_conv.py:145-148)
    if stats is not None:
        # morphology.py:125-128; padded_shape reports the B200 FFT extents: tile + tonal length
        stats["max_abs_deviation"] = max(stats.get("max_abs_deviation", 0.0), dev_max)
        info = plan.info
        tile = (info["tile_x"],) if f.ndim == 1 else (info["tile_y"], info["tile_x"])
        stats["padded_shape"] = tuple(tile) + (info["tonal_len"],)
    if small:
        mn, mx = torch.aminmax(out[0])
        return out[0].to(torch.int64).numpy(), valid[0].to(torch.bool).numpy(), (int(mn), int(mx))
    mn, mx = torch.aminmax(out[0])
    # results come back in the plan's narrow type and widen to the reference's int64 / bool
    # with torch's multithreaded CPU conversions (pinned staging, one copy each)
    o_host = torch.empty(out[0].shape, dtype=out.dtype, pin_memory=True)
    v_host = torch.empty(valid[0].shape, dtype=torch.uint8, pin_memory=True)
    o_host.copy_(out[0], non_blocking=True)
    v_host.copy_(valid[0], non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    values = o_host.to(torch.int64).numpy()
    vmask = v_host.to(torch.bool).numpy()
    return values, vmask, (int(mn), int(mx))


def _empty_crop_quirk(f_ranges, conv_ranges):
    # Reference quirk: with crop=True and F ∩ (F⊕B) empty,
    # intersect_ranges returns None and project_with_validity raises TypeError
    # (morphology.py:132-133 -> umbra.py:193 -> tensor.py:96).  Mirrored for drop-in parity.
    if intersect_ranges(f_ranges, conv_ranges) is None:
        raise TypeError("'NoneType' object is not iterable (image domain and dilation range "
                        "do not intersect; reference dilate_fft raises here)")


# --------------------------------------------------------------------------- FFT path

def dilate_fft(f, b, *, crop: bool = True, return_validity: bool = False,
               stats: dict | None = None):
    """Exact dilation via the tonal lift (morphology.py:116-144), on the GPU."""
    f = GridFunction.coerce(f)
    b = GridFunction.coerce(b)
    if f.ndim != b.ndim:
        raise ValueError("rank mismatch")
    if f.min_defined() < 0 or b.min_defined() < 0:
        raise ValueError("tonal lift needs non-negative values")
    conv = full_output_range(f.ranges, b.ranges)
    if crop:
        _empty_crop_quirk(f.ranges, conv)
    values, valid, rng = _run_fft(f, b, mode="dilate", crop=crop, fill=0, stats=stats)
    out_ranges = f.ranges if crop else conv
    tonal_max = max(f.tonal_max + b.max_defined(), 1)
    g = GridFunction._from_device(values, tuple(lo for lo, _ in out_ranges), tonal_max, False, *rng)
    return (g, valid) if return_validity else g


def reflect(b) -> GridFunction:
    """Index negation about the origin; values and gaps carried along (morphology.py:147-152)."""
    b = GridFunction.coerce(b)
    rev = (slice(None, None, -1),) * b.ndim
    lo = tuple(-hi for hi in b.hi)
    return GridFunction(b.values[rev], b.defined[rev], lo=lo,
                        tonal_max=b.tonal_max, signed=b.signed)


def negate(f, l: int) -> GridFunction:
    """Pointwise l - f(x); gaps preserved (morphology.py:155-163)."""
    f = GridFunction.coerce(f)
    l = int(l)
    if f.min_defined() < 0:
        raise ValueError("cannot negate a grid with negative values")
    if l < f.max_defined():
        raise ValueError(f"l={l} below max value {f.max_defined()}")
    values = np.where(f.defined, l - f.values, np.int64(0))
    return GridFunction(values, f.defined.copy(), lo=f.lo, tonal_max=max(l, 1))


def erode_fft(f, b, l: int | None = None, *, return_validity: bool = False,
              stats: dict | None = None):
    """Erosion by duality, l - dilate_fft(negate(f, l), reflect(b)) (morphology.py:166-180).

    Computed in one GPU pass with l' = max f in place of l (bit-identical at
    valid pixels, shorter tonal axis); pixels with no pair get l."""
    f = GridFunction.coerce(f)
    b = GridFunction.coerce(b)
    if l is None:
        l = f.tonal_max
    l = int(l)
    # negate(f, l) checks (morphology.py:158-161)
    if f.min_defined() < 0:
        raise ValueError("cannot negate a grid with negative values")
    if l < f.max_defined():
        raise ValueError(f"l={l} below max value {f.max_defined()}")
    if f.ndim != b.ndim:
        raise ValueError("rank mismatch")
    # dilate_fft(negate(f), reflect(b)) checks (morphology.py:119-120)
    if b.min_defined() < 0:
        raise ValueError("tonal lift needs non-negative values")
    rb_ranges = tuple((-hi, -lo) for lo, hi in b.ranges)
    _empty_crop_quirk(f.ranges, full_output_range(f.ranges, rb_ranges))
    values, valid, rng = _run_fft(f, b, mode="erode", crop=True, fill=l, stats=stats)
    g = GridFunction._from_device(values, f.lo, max(f.tonal_max, l), True, *rng)
    return (g, valid) if return_validity else g


def _dilate_fft_signed(f, b, **kw):
    """dilate_fft extended to signed inputs by a value shift (morphology.py:198-216).

    The shift is applied inside the encode (v = f - min f) and undone in the
    degree store, so no shifted copy of the image is built."""
    f = GridFunction.coerce(f)
    b = GridFunction.coerce(b)
    m = f.min_defined()
    if m >= 0:
        return dilate_fft(f, b, **kw)
    crop = kw.get("crop", True)
    want_validity = kw.get("return_validity", False)
    stats = kw.get("stats")
    unknown = set(kw) - {"crop", "return_validity", "stats"}
    if unknown:
        raise TypeError(f"unexpected keyword argument {sorted(unknown)[0]!r}")
    if f.ndim != b.ndim:
        raise ValueError("rank mismatch")
    if b.min_defined() < 0:
        raise ValueError("tonal lift needs non-negative values")
    conv = full_output_range(f.ranges, b.ranges)
    if crop:
        _empty_crop_quirk(f.ranges, conv)
    values, valid, rng = _run_fft(f, b, mode="dilate", crop=crop, fill=0, stats=stats)
    out_ranges = f.ranges if crop else conv
    shift = -m
    tonal_max = max(f.tonal_max + shift + b.max_defined(), 1)
    g = GridFunction._from_device(values, tuple(lo for lo, _ in out_ranges), tonal_max, True, *rng)
    return (g, valid) if want_validity else g


# --------------------------------------------------------------------------- direct path

def _naive(f: GridFunction, b: GridFunction, *, mode: str, crop: bool, fill: int):
    dev = _device()
    if f.ndim != b.ndim:
        raise ValueError("rank mismatch")
    if f.ndim not in (1, 2):
        raise NotImplementedError("only 1-D signals and 2-D images are supported")
    bound = max(abs(f.max_defined()), abs(f.min_defined())) + max(abs(b.max_defined()), abs(b.min_defined()))
    if bound >= 2**31:
        raise NotImplementedError("values beyond int32")
    img, mask, _, _, _ = _upload(f, dev)
    out, valid = engine.naive(img=img.unsqueeze(0), defined=None if mask is None else mask.unsqueeze(0),
                              shape=f.shape, se_values=b.values,
                              se_defined=None if b.gap_free else b.defined, se_lo=b.lo,
                              mode=mode, crop=crop, fill=fill)
    return out[0].cpu().to(torch.int64).numpy(), valid[0].cpu().to(torch.bool).numpy()


def dilate_naive(f, b, *, crop: bool = True, return_validity: bool = False):
    """Sliding max of f(x-y)+b(y) over all defined pairs (morphology.py:65-85), GPU direct kernel."""
    f = GridFunction.coerce(f)
    b = GridFunction.coerce(b)
    out_ranges = full_output_range(f.ranges, b.ranges)
    values, valid = _naive(f, b, mode="dilate", crop=crop, fill=0)
    if crop:
        out_ranges = f.ranges
    tonal_max = max(f.tonal_max + b.max_defined(), 1)
    g = GridFunction(values, lo=tuple(lo for lo, _ in out_ranges), tonal_max=tonal_max, signed=f.signed)
    return (g, valid) if return_validity else g


def erode_naive(f, b, *, crop: bool = True, return_validity: bool = False):
    """Sliding min of f(x+y)-b(y); neutral f.tonal_max where no pair exists (morphology.py:88-113)."""
    f = GridFunction.coerce(f)
    b = GridFunction.coerce(b)
    out_ranges = tuple((flo - bhi, fhi - blo) for (flo, fhi), (blo, bhi) in zip(f.ranges, b.ranges))
    values, valid = _naive(f, b, mode="erode", crop=crop, fill=f.tonal_max)
    if crop:
        out_ranges = f.ranges
    g = GridFunction(values, lo=tuple(lo for lo, _ in out_ranges), tonal_max=f.tonal_max, signed=True)
    return (g, valid) if return_validity else g


# --------------------------------------------------------------------------- dispatch + compound

def dilate(f, b, method=MorphMethod.NAIVE, **kw):
    """morphology.py:183-187."""
    method = MorphMethod.parse(method)
    if method is MorphMethod.NAIVE:
        return dilate_naive(f, b, **kw)
    return _dilate_fft_signed(f, b, **kw)


def erode(f, b, method=MorphMethod.NAIVE, l: int | None = None, **kw):
    """morphology.py:190-195."""
    method = MorphMethod.parse(method)
    if method is MorphMethod.NAIVE:
        return erode_naive(f, b, **kw)
    return erode_fft(f, b, l=l, **kw)


def opening(f, b, method=MorphMethod.NAIVE, l: int | None = None,
            stats: dict | None = None) -> GridFunction:
    """morphology.py:219-222."""
    kw = {} if MorphMethod.parse(method) is MorphMethod.NAIVE else {"stats": stats}
    return dilate(erode(f, b, method, l=l, **kw), b, method, **kw)


def closing(f, b, method=MorphMethod.NAIVE, l: int | None = None,
            stats: dict | None = None) -> GridFunction:
    """morphology.py:225-229."""
    kw = {} if MorphMethod.parse(method) is MorphMethod.NAIVE else {"stats": stats}
    d = dilate(f, b, method, **kw)
    return erode(d, b, method, l=d.tonal_max if l is None else l, **kw)


def beucher_gradient(f, b, method=MorphMethod.NAIVE, l: int | None = None,
                     stats: dict | None = None) -> GridFunction:
    """morphology.py:232-239."""
    kw = {} if MorphMethod.parse(method) is MorphMethod.NAIVE else {"stats": stats}
    d = dilate(f, b, method, **kw)
    e = erode(f, b, method, l=l, **kw)
    values = np.maximum(d.values - e.values, np.int64(0))
    return GridFunction(values, lo=GridFunction.coerce(f).lo,
                        tonal_max=max(int(values.max()), 1))
