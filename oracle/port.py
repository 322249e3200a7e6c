"""ORACLE — test infrastructure only.  Never imported by the product package.

CPU restatement (numpy / scipy) of the reference's hot path, used as the
checker by tests/, by __graft_entry__.smoke() and as the ``cpu_baseline`` /
``--impl reference`` arm of bench.py.  Every function cites the reference
lines it restates (reference = fftmorph 0.1.0 under /root/reference/pkg/src,
not vendored here).

Pinned: tests/test_oracle.py checks these functions against the reference's
own golden vectors (conftest.py:10-61, test_morphology.py, test_umbra.py) and
against fixtures produced by running the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz).

Grids are passed as plain arrays: ``values`` (int), ``defined`` (bool or
None = all defined) and ``lo`` (tuple of logical origins).
"""

from __future__ import annotations

import numpy as np
import scipy.fft

BIG = np.int64(1) << 40          # morphology.py:27
MAX_DEVIATION = 0.25             # fft_conv.py:22
PRECISION_BUDGET = 2 ** 52       # fft_conv.py:19


def _ranges(shape, lo):
    return tuple((int(l), int(l) + int(n) - 1) for l, n in zip(lo, shape))


def full_output_range(ra, rb):
    """tensor.py:76-89."""
    return tuple((la + lb, ha + hb) for (la, ha), (lb, hb) in zip(ra, rb))


def intersect_ranges(ra, rb):
    """tensor.py:92-101."""
    out = []
    for (la, ha), (lb, hb) in zip(ra, rb):
        lo, hi = max(la, lb), min(ha, hb)
        if hi < lo:
            return None
        out.append((lo, hi))
    return tuple(out)


def paste(f_ranges, src, src_ranges, fill):
    """morphology.py:51-62."""
    shape = tuple(hi - lo + 1 for lo, hi in f_ranges)
    out = np.full(shape, fill, dtype=src.dtype)
    inter = intersect_ranges(f_ranges, src_ranges)
    if inter is not None:
        dst = tuple(slice(lo - flo, hi - flo + 1) for (lo, hi), (flo, _) in zip(inter, f_ranges))
        srcs = tuple(slice(lo - slo, hi - slo + 1) for (lo, hi), (slo, _) in zip(inter, src_ranges))
        out[dst] = src[srcs]
    return out


def _prep(values, defined):
    v = np.asarray(values, dtype=np.int64)
    d = np.ones(v.shape, bool) if defined is None else np.asarray(defined, bool)
    return v, d


def dilate_naive(f, f_def, f_lo, b, b_def, b_lo, *, crop=True):
    """Sliding max of f(x-y)+b(y) over defined pairs (morphology.py:65-85).
    Returns (values int64, valid bool, out_lo)."""
    f, f_def = _prep(f, f_def)
    b, b_def = _prep(b, b_def)
    fr, br = _ranges(f.shape, f_lo), _ranges(b.shape, b_lo)
    out_ranges = full_output_range(fr, br)
    acc = np.full(tuple(h - l + 1 for l, h in out_ranges), -BIG, dtype=np.int64)
    fv = np.where(f_def, f, -BIG)
    for idx in np.argwhere(b_def):
        w = b[tuple(idx)]
        sl = tuple(slice(i, i + n) for i, n in zip(idx, f.shape))
        np.maximum(acc[sl], fv + w, out=acc[sl])
    valid = acc > -(BIG >> 1)
    values = np.where(valid, acc, np.int64(0))
    if crop:
        values = paste(fr, values, out_ranges, np.int64(0))
        valid = paste(fr, valid, out_ranges, False)
        out_ranges = fr
    return values, valid, tuple(lo for lo, _ in out_ranges)


def erode_naive(f, f_def, f_lo, b, b_def, b_lo, *, crop=True, neutral):
    """Sliding min of f(x+y)-b(y); neutral where no pair (morphology.py:88-113).
    ``neutral`` is the reference's f.tonal_max."""
    f, f_def = _prep(f, f_def)
    b, b_def = _prep(b, b_def)
    fr, br = _ranges(f.shape, f_lo), _ranges(b.shape, b_lo)
    out_ranges = tuple((flo - bhi, fhi - blo) for (flo, fhi), (blo, bhi) in zip(fr, br))
    acc = np.full(tuple(h - l + 1 for l, h in out_ranges), BIG, dtype=np.int64)
    fv = np.where(f_def, f, BIG)
    for idx in np.argwhere(b_def):
        w = b[tuple(idx)]
        off = tuple(bhi - (blo + i) for i, (blo, bhi) in zip(idx, br))
        sl = tuple(slice(o, o + n) for o, n in zip(off, f.shape))
        np.minimum(acc[sl], fv - w, out=acc[sl])
    valid = acc < (BIG >> 1)
    values = np.where(valid, acc, np.int64(neutral))
    if crop:
        values = paste(fr, values, out_ranges, np.int64(neutral))
        valid = paste(fr, valid, out_ranges, False)
        out_ranges = fr
    return values, valid, tuple(lo for lo, _ in out_ranges)


def next_fast_size(n):
    """fft_conv.py:61-77: smallest of 2^k and 45*2^k that is >= n."""
    pow2 = 1
    while pow2 < n:
        pow2 *= 2
    alt = 45
    while alt < n:
        alt *= 2
    return min(pow2, alt)


def build_umbra(values, defined, l_r):
    """umbra.py:177-186: int64 one-hot volume, tonal axis last."""
    v, d = _prep(values, defined)
    bits = np.zeros(v.shape + (l_r + 1,), dtype=np.int64)
    where = np.nonzero(d)
    bits[where + (v[where],)] = 1
    return bits


def conv_full_fft(a, b, workers=1):
    """fft_conv.py:128-150 (plan fft_conv.py:80-91): real FFT convolution at
    next_fast_size per axis, rint, deviation check.  Returns (counts, dev, padded)."""
    padded = tuple(next_fast_size(sa + sb - 1) for sa, sb in zip(a.shape, b.shape))
    out_shape = tuple(sa + sb - 1 for sa, sb in zip(a.shape, b.shape))
    fa = scipy.fft.rfftn(a.astype(np.float64), s=padded, workers=workers)
    fb = scipy.fft.rfftn(b.astype(np.float64), s=padded, workers=workers)
    fa *= fb
    del fb
    full = scipy.fft.irfftn(fa, s=padded, workers=workers)
    del fa
    sliced = full[tuple(slice(0, n) for n in out_shape)]
    rounded = np.rint(sliced)
    dev = float(np.abs(sliced - rounded).max())
    if dev >= MAX_DEVIATION:
        raise ArithmeticError(f"pre-rounding deviation {dev:.3g} >= {MAX_DEVIATION}")
    return rounded.astype(np.int64), dev, padded


def project_with_validity(counts, counts_lo, out_range):
    """umbra.py:189-205: top nonzero tonal index per pixel over out_range."""
    spatial = tuple((lo, lo + n - 1) for lo, n in zip(counts_lo, counts.shape[:-1]))
    sl = tuple(slice(lo - clo, hi - clo + 1) for (lo, hi), (clo, _) in zip(out_range, spatial))
    window = counts[sl]
    nonzero = window >= 1
    has_any = nonzero.any(axis=-1)
    t = window.shape[-1]
    top = t - 1 - np.argmax(nonzero[..., ::-1], axis=-1)
    return np.where(has_any, top, 0).astype(np.int64), has_any


def dilate_fft(f, f_def, f_lo, b, b_def, b_lo, *, crop=True, workers=1):
    """morphology.py:116-144: tonal lift -> FFT convolution -> projection.
    Returns (values, valid, out_lo, max_abs_deviation, padded_shape)."""
    f, f_def = _prep(f, f_def)
    b, b_def = _prep(b, b_def)
    if f[f_def].min() < 0 or b[b_def].min() < 0:
        raise ValueError("tonal lift needs non-negative values")
    l_r = int(f[f_def].max()) + int(b[b_def].max())          # umbra.py:172-174
    fu = build_umbra(f, f_def, l_r)
    bu = build_umbra(b, b_def, l_r)
    counts, dev, padded = conv_full_fft(fu, bu, workers=workers)
    fr, br = _ranges(f.shape, f_lo), _ranges(b.shape, b_lo)
    conv_spatial = full_output_range(fr, br)
    counts_lo = tuple(lo for lo, _ in conv_spatial)
    if crop:
        inter = intersect_ranges(fr, conv_spatial)
        if inter is None:
            raise TypeError("image domain and dilation range do not intersect (reference quirk)")
        proj, mask = project_with_validity(counts, counts_lo, inter)
        values = paste(fr, proj, inter, np.int64(0))
        valid = paste(fr, mask, inter, False)
        out_lo = tuple(lo for lo, _ in fr)
    else:
        values, valid = project_with_validity(counts, counts_lo, conv_spatial)
        out_lo = counts_lo
    return values, valid, out_lo, dev, padded


def erode_fft(f, f_def, f_lo, b, b_def, b_lo, *, l, workers=1):
    """morphology.py:166-180: l - dilate_fft(negate(f, l), reflect(b)); invalid -> l."""
    f, f_def = _prep(f, f_def)
    b, b_def = _prep(b, b_def)
    if f[f_def].min() < 0:
        raise ValueError("cannot negate a grid with negative values")
    if l < f[f_def].max():
        raise ValueError(f"l={l} below max value")
    neg = np.where(f_def, l - f, 0)                                   # morphology.py:162
    rev = (slice(None, None, -1),) * b.ndim
    rb, rbd = b[rev], b_def[rev]                                      # morphology.py:149-151
    rlo = tuple(-(lo + n - 1) for lo, n in zip(b_lo, b.shape))
    d, valid, out_lo, dev, padded = dilate_fft(neg, f_def, f_lo, rb, rbd, rlo, crop=True, workers=workers)
    return l - d, valid, out_lo, dev, padded
