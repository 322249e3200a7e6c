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
    """Generic operands: the FP64 FFT path (fm_conv_full_fft64) against exact int64 sums."""
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


# ---------------------------------------------------------------- FP64 FFT path (fm_conv_full_fft64)
def _launches():
    from paper_2305_03018_b200 import _lib
    return _lib.kernel_launches()


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_generic_operands_take_the_fp64_fft(ndim):
    """Generic (non one-hot) operands run FFTs on the device, not the direct kernel: the
    radix-pass launches are counted, and the padded shape is the reference's ladder."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats, next_fast_size
    rng = np.random.default_rng(5 + ndim)
    a = OffsetArray(rng.integers(0, 16, (7,) * ndim), (1,) * ndim)
    b = OffsetArray(rng.integers(0, 16, (5,) * ndim), (-2,) * ndim)
    l0 = _launches()
    out, stats = conv_full_fft_with_stats(a, b)
    assert _launches() - l0 >= 3 * ndim     # >= one radix pass per axis for each of 3 transforms
    assert stats.padded_shape == tuple(next_fast_size(11) for _ in range(ndim))
    assert np.array_equal(out.data, _np_full(a.data, b.data))
    assert 0.0 <= stats.max_abs_deviation < 1e-9      # FP64 on small integers


def test_fp64_large_values_and_45_ladder():
    """Magnitudes near the reference's scale (2^20 values) and a 45*2^k padded length."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats
    rng = np.random.default_rng(77)
    a = OffsetArray(rng.integers(0, 1 << 20, 60))
    b = OffsetArray(rng.integers(0, 1 << 10, 30))     # full length 89 -> padded 90 = 45*2
    out, stats = conv_full_fft_with_stats(a, b)
    assert stats.padded_shape == (90,)
    assert np.array_equal(out.data, _np_full(a.data, b.data))
    assert stats.max_abs_deviation < 0.25


def test_fft_delta_commutative_bilinear():
    """test_fft_conv.py TestFft semantics: delta identity, commutativity, bilinearity."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft
    a = OffsetArray(np.arange(24).reshape(4, 6), lo=(-2, 1))
    out = conv_full_fft(a, OffsetArray(np.array([[1]]), lo=(0, 0)))
    assert out.lo == a.lo and np.array_equal(out.data, a.data)
    rng = np.random.default_rng(5)
    x = OffsetArray(rng.integers(0, 16, (5, 7)), (1, -3))
    y = OffsetArray(rng.integers(0, 16, (4, 2)), (0, 2))
    p, q = conv_full_fft(x, y), conv_full_fft(y, x)
    assert p.lo == q.lo and np.array_equal(p.data, q.data)
    a1 = OffsetArray(rng.integers(0, 16, 6))
    a2 = OffsetArray(rng.integers(0, 16, 6))
    bb = OffsetArray(rng.integers(0, 16, 4))
    lhs = conv_full_fft(OffsetArray(a1.data + a2.data), bb).data
    assert np.array_equal(lhs, conv_full_fft(a1, bb).data + conv_full_fft(a2, bb).data)


def test_precision_budget_violation():
    """fft_conv.py:114-125 (test_fft_conv.py test_precision_budget_violation)."""
    import paper_2305_03018_b200 as m
    a = m.OffsetArray(np.full(32, 1 << 32))
    with pytest.raises(m.PrecisionBudgetError):
        m.conv_full_fft(a, a)


def test_transforms_zero_roundtrip_theorem():
    """test_fft_conv.py TestTransforms semantics on the device FP64 DFT (fm_fft64)."""
    import paper_2305_03018_b200 as m
    plan = m.make_plan(m.OffsetArray(np.zeros(5, np.int64)), m.OffsetArray(np.zeros(4, np.int64)), m.Backend.FFT)
    assert not m.transform_forward(np.zeros(5), plan).any()
    rng = np.random.default_rng(31)
    a = rng.integers(0, 1 << 20, (7, 9)).astype(np.float64)
    plan = m.make_plan(m.OffsetArray(a.astype(np.int64)), m.OffsetArray(np.ones((3, 3), np.int64)), m.Backend.FFT)
    spec = m.transform_forward(a, plan)
    assert np.allclose(spec, np.fft.fftn(a, s=plan.padded_shape, axes=(0, 1)), rtol=1e-12, atol=1e-6)
    back = m.transform_inverse(spec, plan)
    sl = tuple(slice(0, n) for n in a.shape)
    assert np.abs(back[sl].real - a).max() / a.max() < 1e-9
    x = m.OffsetArray(rng.integers(0, 16, (5, 6)))
    y = m.OffsetArray(rng.integers(0, 16, (4, 3)))
    plan = m.make_plan(x, y, m.Backend.FFT)
    prod = m.transform_forward(x.data.astype(float), plan) * m.transform_forward(y.data.astype(float), plan)
    back = m.transform_inverse(prod, plan)
    got = np.rint(back[:8, :8].real).astype(np.int64)
    assert np.array_equal(got, m.conv_full_direct(x, y).data)


def test_umbra_of_3d_grids_through_fp64():
    """Umbra volumes of 3-D grids (rank-4 arrays) have no tile path: FP64 FFT, exact."""
    from paper_2305_03018_b200.fft_conv import OffsetArray, conv_full_fft_with_stats
    rng = np.random.default_rng(8)
    fv = rng.integers(0, 5, (4, 3, 5))
    bv = rng.integers(0, 3, (2, 2, 2))
    fu = port.build_umbra(fv, None, 7)
    bu = port.build_umbra(bv, None, 7)
    out, stats = conv_full_fft_with_stats(OffsetArray(fu), OffsetArray(bu))
    assert np.array_equal(out.data, _np_full(fu, bu))


def test_fp32_count_budget_raises_precision_error():
    """a-priori FP32 budget of the hot path (fm_plan_desc.count_budget): a 15x15 flat SE
    can reach 225 pairs per degree; with a budget of 100 the plan refuses."""
    import torch
    import paper_2305_03018_b200 as m
    from paper_2305_03018_b200.engine import MorphPlan
    with pytest.raises(m.PrecisionBudgetError):
        MorphPlan(shape=(64, 64), se_values=np.zeros((15, 15), np.int64), se_lo=(-7, -7), img_min=0,
                  img_max=31, device=torch.device("cuda", 0), count_budget=100)
    p = MorphPlan(shape=(64, 64), se_values=np.zeros((15, 15), np.int64), se_lo=(-7, -7), img_min=0,
                  img_max=31, device=torch.device("cuda", 0), count_budget=226)
    p.close()


# ---------------------------------------------------------------- count-level types (umbra.py)
IMAGE_LIFT = [[0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 0], [0, 0, 1, 0, 0, 1], [0, 0, 0, 1, 0, 0],
              [0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 0, 0], [1, 0, 0, 0, 0, 0], [0, 0, 0, 0, 1, 0],
              [0, 0, 0, 0, 0, 0], [0, 1, 0, 0, 0, 0]]
SE_LIFT = [[0, 0, 0, 0]] * 7 + [[0, 1, 0, 0], [1, 0, 0, 0], [0, 0, 0, 1]]


def _bits(matrix):
    return np.asarray(matrix, dtype=np.int64)[::-1].T.copy()


def test_build_umbra_matrices(example_image, example_se):
    """test_umbra.py TestBuildUmbra semantics, on the device (fm_build_umbra)."""
    import paper_2305_03018_b200 as m
    u = m.build_umbra(example_image, 9)
    assert u.bits.lo == (0, 0) and np.array_equal(u.bits.data, _bits(IMAGE_LIFT))
    s = m.build_umbra(example_se, 9)
    assert s.bits.lo == (-1, 0) and np.array_equal(s.bits.data, _bits(SE_LIFT))
    assert not s.bits.data[2].any()
    z = m.build_umbra(m.GridFunction(np.zeros((2, 3), np.int64), tonal_max=1), 0)
    assert z.bits.data.shape == (2, 3, 1) and z.bits.data.all()
    with pytest.raises(ValueError):
        m.build_umbra(example_image, 6)
    rng = np.random.default_rng(2)
    g = m.GridFunction(rng.integers(0, 8, (5, 7)), rng.random((5, 7)) < 0.8, tonal_max=7)
    u = m.build_umbra(g, 10)
    u.verify()
    assert set(np.unique(u.bits.data.sum(axis=-1))) <= {0, 1}
    assert u.bits.data.sum() == g.defined.sum()


def test_required_lr_and_project(example_image, example_se):
    """test_umbra.py TestRequiredLr / TestProject semantics (fm_project on the device)."""
    import paper_2305_03018_b200 as m
    assert m.required_lr(example_image, example_se) == 9
    z = m.GridFunction(np.zeros(4, np.int64), tonal_max=1)
    assert m.required_lr(z, z) == 0
    c = m.CountVolume(m.OffsetArray(_bits(RESULT_COUNT_MATRIX), (0, 0)), 9)
    assert m.project(c, ((0, 5),)).to_list() == [5, 8, 9, 8, 8, 9]
    c0 = m.CountVolume(m.OffsetArray(np.zeros((4, 6), np.int64)), 5)
    g, valid = m.project_with_validity(c0, ((0, 3),))
    assert not g.values.any() and not valid.any()
    col = np.zeros((1, 10), np.int64)
    col[0, [3, 7, 9]] = 1
    assert m.project(m.CountVolume(m.OffsetArray(col, (2, 0)), 9), ((2, 2),)).to_list() == [9]
    with pytest.raises(ValueError):
        m.project(c0, ((0, 4),))


def test_pipeline_volume(example_image, example_se):
    """test_umbra.py TestPipelineVolume: worked-example counts, round trip, pair enumeration."""
    import paper_2305_03018_b200 as m
    fu, bu = m.build_umbra(example_image, 9), m.build_umbra(example_se, 9)
    counts = m.conv_full_fft(fu.bits, bu.bits)
    vol = m.CountVolume(counts, 9)
    vol.verify()
    assert np.array_equal(counts.data[1:7, :10], _bits(RESULT_COUNT_MATRIX))
    rng = np.random.default_rng(17)
    g = m.GridFunction(rng.integers(0, 12, (6, 5)), lo=(-2, 1), tonal_max=11)
    assert m.project(m.CountVolume(m.build_umbra(g, 15).bits, 15), g.ranges) == g
    rng = np.random.default_rng(19)
    f = m.GridFunction(rng.integers(0, 6, 7), rng.random(7) < 0.8, lo=(0,), tonal_max=5)
    b = m.GridFunction(rng.integers(0, 4, 4), rng.random(4) < 0.8, lo=(-1,), tonal_max=3)
    l_r = m.required_lr(f, b)
    counts = m.conv_full_fft(m.build_umbra(f, l_r).bits, m.build_umbra(b, l_r).bits)
    for x in range(counts.lo[0], counts.hi[0] + 1):
        for y in range(counts.lo[1], counts.hi[1] + 1):
            exp = 0
            for yy in range(b.lo[0], b.hi[0] + 1):
                xx = x - yy
                if f.lo[0] <= xx <= f.hi[0]:
                    fv, bv = f.at((xx,)), b.at((yy,))
                    if fv is not None and bv is not None and fv + bv == y:
                        exp += 1
            assert counts.at((x, y)) == exp
