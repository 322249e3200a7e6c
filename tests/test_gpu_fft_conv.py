"""GPU: the count-level API (fft_conv.py of the reference) against exact int64 oracles.

Mirrors test_fft_conv.py:39-114 and test_umbra.py:85-123: direct GPU convolution
of generic integer arrays, and umbra count volumes through the FFT tile path in
count-volume mode (FM_FLAG_COUNTS), both bit-exact."""

import numpy as np
import pytest

from conftest import RESULT_COUNT_MATRIX
from oracle import port

pytestmark = pytest.mark.gpu


def _np_full(a, b):
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    out = np.zeros(tuple(x + y - 1 for x, y in zip(a.shape, b.shape)), np.int64)
    for idx in np.ndindex(*b.shape):
        if b[idx]:
            out[tuple(slice(i, i + n) for i, n in zip(idx, a.shape))] += b[idx] * a
    return out


def test_direct_binomial_monomial_zero():
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_direct, direct_full
    out = conv_full_direct(OffsetArray(np.array([1, 1])), OffsetArray(np.array([1, 1])))
    assert out.lo == (0,) and out.data.tolist() == [1, 2, 1]
    a = np.zeros(10, np.int64)
    a[3] = 1
    b = np.zeros(10, np.int64)
    b[0] = 1
    exp = np.zeros(19, np.int64)
    exp[3] = 1
    assert np.array_equal(direct_full(a, b), exp)
    z = conv_full_direct(OffsetArray(np.arange(1, 7).reshape(2, 3)), OffsetArray(np.zeros((2, 2), np.int64)))
    assert not z.data.any()


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_fft_matches_direct_randomized(ndim):
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats
    rng = np.random.default_rng(23 + ndim)
    for _ in range(30):
        def one():
            shape = tuple(int(e) for e in rng.integers(1, 10, ndim))
            lo = tuple(int(x) for x in rng.integers(-4, 5, ndim))
            return OffsetArray(rng.integers(0, 16, shape), lo)
        a, b = one(), one()
        fast, stats = conv_full_fft_with_stats(a, b)
        assert fast.lo == tuple(x + y for x, y in zip(a.lo, b.lo))
        assert np.array_equal(fast.data, _np_full(a.data, b.data))
        assert stats.max_abs_deviation < 0.25


def test_umbra_worked_example_counts(example_image, example_se):
    """test_umbra.py:85-94: count matrix of the worked example through the FFT path."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats
    f, b = example_image, example_se
    fu = port.build_umbra(f.values, f.defined, 9)
    bu = port.build_umbra(b.values, b.defined, 9)
    counts, stats = conv_full_fft_with_stats(OffsetArray(fu, f.lo + (0,)), OffsetArray(bu, b.lo + (0,)))
    window = counts.data[1:7, :10]
    expected = np.array(RESULT_COUNT_MATRIX)[::-1].T      # rows 9..0 -> degrees 0..9
    assert np.array_equal(window, expected)
    assert stats.max_abs_deviation < 0.25


@pytest.mark.parametrize("ndim", [1, 2])
def test_umbra_counts_match_exact(ndim):
    """Umbra count volumes (test_umbra.py:96-123 semantics) vs exact int64 convolution,
    with gaps, arbitrary origins and tonal extents."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats
    rng = np.random.default_rng(19 + ndim)
    for trial in range(12):
        fs = tuple(int(x) for x in rng.integers(2, 40 if ndim == 2 else 300, ndim))
        bs = tuple(int(x) for x in rng.integers(1, 9, ndim))
        fmax, bmax = int(rng.integers(1, 40)), int(rng.integers(0, 12))
        fv = rng.integers(0, fmax + 1, fs)
        fd = rng.random(fs) < 0.85
        bv = rng.integers(0, bmax + 1, bs)
        bd = rng.random(bs) < 0.8
        if not fd.any() or not bd.any():
            continue
        l_r = fmax + bmax
        fu = port.build_umbra(fv, fd, l_r)
        bu = port.build_umbra(bv, bd, l_r)
        flo = tuple(int(x) for x in rng.integers(-5, 5, ndim)) + (0,)
        blo = tuple(int(x) for x in rng.integers(-5, 5, ndim)) + (0,)
        counts, stats = conv_full_fft_with_stats(OffsetArray(fu, flo), OffsetArray(bu, blo))
        assert counts.lo == tuple(x + y for x, y in zip(flo, blo))
        assert np.array_equal(counts.data, _np_full(fu, bu)), trial
        assert stats.max_abs_deviation < 0.25
