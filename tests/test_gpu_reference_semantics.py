"""GPU: the rest of the reference test-suite's semantics through the drop-in API.

Restated from the reference's own tests (our inputs and code, same properties):
dilate_naive / erode_naive (test_morphology.py:33-100: identity and flat SEs,
monotonicity, extensivity, translation covariance, validity mask, constant
images, negative erosion), the FFT path's histogram equality with the direct
method (test_morphology.py:131-137), and the acceptance criteria 2 (exactness
sweep over sizes, bit depths and SE widths) and 7 (duality, the open/close
sandwich, histogram equality) of test_acceptance.py:69-108,200-221 -- all
running on the B200 (`method="naive"` is the GPU direct kernel).
"""

import numpy as np
import pytest

from conftest import flat_se, identity_se, random_grid

pytestmark = pytest.mark.gpu


def M():
    import paper_2305_03018_b200 as m
    return m


class TestDilateNaive:
    def test_identity_and_flat(self, example_image):
        assert M().dilate_naive(example_image, identity_se()) == example_image
        assert M().dilate_naive(example_image, flat_se(3)).to_list() == [3, 7, 7, 7, 7, 7]

    def test_monotone(self):
        rng = np.random.default_rng(141)
        f = random_grid(rng, (8, 8), 14)
        g = M().GridFunction(f.values + rng.integers(0, 2, f.shape), tonal_max=16)
        b = random_grid(rng, (3, 3), 5, lo=(-1, -1))
        for fn in (M().dilate_naive, M().dilate_fft):
            assert (fn(f, b).values <= fn(g, b).values).all()

    def test_extensive_when_origin_defined(self):
        rng = np.random.default_rng(143)
        f = random_grid(rng, (9, 7), 10)
        b = random_grid(rng, (3, 3), 4, lo=(-1, -1))
        b = M().GridFunction(b.values, np.ones_like(b.defined), lo=b.lo, tonal_max=b.tonal_max)
        for fn in (M().dilate_naive, M().dilate_fft):
            assert (fn(f, b).values >= f.values + b.at((0, 0))).all()

    def test_translation_covariance_uncropped(self):
        rng = np.random.default_rng(147)
        f = random_grid(rng, (6,), 9)
        b = random_grid(rng, (4,), 5, lo=(-1,))
        shifted = M().GridFunction(b.values, b.defined, lo=(b.lo[0] + 3,), tonal_max=b.tonal_max)
        for fn in (M().dilate_naive, M().dilate_fft):
            out, out_s = fn(f, b, crop=False), fn(f, shifted, crop=False)
            assert out_s.lo == (out.lo[0] + 3,)
            assert np.array_equal(out.values, out_s.values)

    def test_validity_mask_far_se(self):
        f = M().GridFunction(np.array([1, 2]), tonal_max=3)
        b = M().GridFunction(np.array([0]), lo=(5,), tonal_max=1)
        out, valid = M().dilate_naive(f, b, return_validity=True)
        assert not valid.any() and not out.values.any()


class TestErodeNaive:
    def test_flat_identity_constant(self, example_image):
        assert M().erode_naive(example_image, flat_se(3)).to_list() == [0, 0, 0, 2, 2, 2]
        assert M().erode_naive(example_image, identity_se()) == example_image
        c = M().GridFunction(np.full((4, 4), 6), tonal_max=9)
        assert (M().erode_naive(c, flat_se(3, ndim=2)).values == 6).all()
        assert (M().erode_fft(c, flat_se(3, ndim=2)).values == 6).all()

    def test_can_go_negative(self):
        f = M().GridFunction(np.array([0, 0, 0]), tonal_max=5)
        b = M().GridFunction(np.array([3]), lo=(0,), tonal_max=3)
        assert M().erode_naive(f, b).to_list() == [-3, -3, -3]
        assert M().erode_fft(f, b).to_list() == [-3, -3, -3]


def test_histogram_equality():
    from paper_2305_03018_b200.pgmio import histogram
    rng = np.random.default_rng(161)
    f = random_grid(rng, (32, 32), 15)
    b = flat_se(5, ndim=2)
    assert np.array_equal(histogram(M().dilate_fft(f, b)), histogram(M().dilate_naive(f, b)))


def test_acceptance_exactness_sweep():
    """Criterion 2 semantics: FFT == direct (values and validity) over image sizes, bit
    depths 1..8, flat and non-flat SEs of several widths, with gaps."""
    rng = np.random.default_rng(2000)
    runs = 0
    for bits in (1, 2, 4, 6, 8):
        top = (1 << bits) - 1
        for edge in (7, 33, 64, 130):
            for fe in (1, 3, 5, 9, 17):
                if fe > edge:
                    continue
                f = random_grid(rng, (edge, edge), top, gap_p=0.1 if runs % 3 == 0 else 0.0)
                sev = rng.integers(0, top + 1, (fe, fe)) if runs % 2 else np.zeros((fe, fe), np.int64)
                b = M().GridFunction(sev, lo=(-(fe // 2), -(fe // 2)), tonal_max=max(top, 1))
                d, dv = M().dilate_fft(f, b, return_validity=True)
                n, nv = M().dilate_naive(f, b, return_validity=True)
                assert d == n and np.array_equal(dv, nv), (bits, edge, fe)
                e, ev = M().erode_fft(f, b, return_validity=True)
                en, env = M().erode_naive(f, b, return_validity=True)
                assert np.array_equal(ev, env)
                assert np.array_equal(e.values[ev], en.values[env])
                runs += 1
    assert runs > 60


def test_acceptance_morphology_algebra():
    """Criterion 7 semantics on 20 random 64x64 images: erosion duality in the interior,
    opening <= f <= closing, histogram equality of the FFT and direct dilations."""
    from paper_2305_03018_b200.pgmio import histogram
    rng = np.random.default_rng(7001)
    b = flat_se(5, ndim=2)
    inner = (slice(2, -2), slice(2, -2))
    for _ in range(20):
        f = M().GridFunction(rng.integers(0, 16, (64, 64)), tonal_max=15)
        assert np.array_equal(M().erode_fft(f, b).values[inner], M().erode_naive(f, b).values[inner])
        o = M().opening(f, b, M().MorphMethod.FFT_UMBRA)
        c = M().closing(f, b, M().MorphMethod.FFT_UMBRA)
        assert (o.values[inner] <= f.values[inner]).all()
        assert (f.values[inner] <= c.values[inner]).all()
        assert np.array_equal(histogram(M().dilate_fft(f, b)), histogram(M().dilate_naive(f, b)))
