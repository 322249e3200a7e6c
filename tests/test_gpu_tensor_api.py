"""GPU: batched device API and on-device compound operators."""

import numpy as np
import pytest

from oracle import cnaive, port

pytestmark = pytest.mark.gpu


def _ref_erode(img, se, lo, l):
    v, _ = cnaive.naive(img, None, se, None, lo, erode=True, fill=l)
    return v.astype(np.int64)


def _ref_dilate(img, se, lo):
    v, _ = cnaive.naive(img, None, se, None, lo)
    return v.astype(np.int64)


def test_dilate_erode_batch_and_single():
    import torch
    from paper_2305_03018_b200 import tensor_api as TA
    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 50, (4, 64, 80)).astype(np.uint8)
    se = rng.integers(0, 7, (5, 7))
    x = torch.from_numpy(imgs).cuda()
    d, dv = TA.dilate(x, se)
    e, ev = TA.erode(x, se)
    d1, _ = TA.dilate(x[2], se)
    for i in range(4):
        assert np.array_equal(d[i].cpu().numpy(), _ref_dilate(imgs[i], se, (-2, -3)))
        assert np.array_equal(e[i].cpu().numpy(), _ref_erode(imgs[i], se, (-2, -3), int(imgs.max())))
    assert np.array_equal(d1.cpu().numpy(), d[2].cpu().numpy())
    assert dv.all() and ev.all()


def test_compound_on_device_match_oracle():
    import torch
    from paper_2305_03018_b200 import tensor_api as TA
    rng = np.random.default_rng(5)
    img = rng.integers(0, 16, (48, 40)).astype(np.uint8)
    se = rng.integers(0, 5, (5, 5))
    lo = (-2, -2)
    x = torch.from_numpy(img).cuda()
    hi = int(img.max())
    e = _ref_erode(img, se, lo, hi)
    opening_ref = _ref_dilate(e - e.min(), se, lo) + e.min()     # dilation commutes with shifts
    assert np.array_equal(TA.opening(x, se, lo).cpu().numpy(), opening_ref)
    d = _ref_dilate(img, se, lo)
    closing_ref = _ref_erode(d, se, lo, hi + int(se.max()))
    assert np.array_equal(TA.closing(x, se, lo).cpu().numpy(), closing_ref)
    grad_ref = np.maximum(d - _ref_erode(img, se, lo, hi), 0)
    assert np.array_equal(TA.gradient(x, se, lo).cpu().numpy(), grad_ref)


def test_device_api_matches_dropin_compound():
    """On-device opening/closing/gradient equal the GridFunction API (reference semantics)
    when every pixel has a pair (centred SE) and tonal_max is the data maximum."""
    import torch
    import paper_2305_03018_b200 as fm
    from paper_2305_03018_b200 import tensor_api as TA
    rng = np.random.default_rng(9)
    img = rng.integers(0, 30, (33, 47))
    se = rng.integers(0, 4, (3, 5))
    f = fm.GridFunction(img, tonal_max=int(img.max()))
    b = fm.GridFunction(se, lo=(-1, -2), tonal_max=max(int(se.max()), 1))
    x = torch.from_numpy(img.astype(np.uint8)).cuda()
    assert np.array_equal(TA.opening(x, se, (-1, -2)).cpu().numpy(), fm.opening(f, b, "fft").values)
    assert np.array_equal(TA.closing(x, se, (-1, -2)).cpu().numpy(), fm.closing(f, b, "fft").values)
    assert np.array_equal(TA.gradient(x, se, (-1, -2)).cpu().numpy(), fm.beucher_gradient(f, b, "fft").values)
