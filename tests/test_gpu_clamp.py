"""GPU: the per-unit clamp bound of fm_range.cuh (values below D - max b encode as the clamp).

The clamp is exact by construction (tests/test_oracle.py checks the integer
model); these tests check the CUDA path against the C oracle on inputs where
it fires hard (smooth images, flat SEs with random masks, gaps, crop off,
erosion), and that it really reduces the planes computed.
"""

import os
import zlib

import numpy as np
import pytest

from oracle import cnaive

pytestmark = pytest.mark.gpu


def _smooth(rng, shape, levels):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(rng.standard_normal(shape), 3.0)
    x = (x - x.min()) / (x.max() - x.min())
    return np.rint(x * (levels - 1)).astype(np.uint8)


def _plan(taps, **kw):
    from paper_2305_03018_b200.engine import MorphPlan
    old = os.environ.get("FM_RANGE_TAPS")
    os.environ["FM_RANGE_TAPS"] = str(taps)
    try:
        return MorphPlan(**kw)
    finally:
        if old is None:
            del os.environ["FM_RANGE_TAPS"]
        else:
            os.environ["FM_RANGE_TAPS"] = old


def _run(taps, imgs, defined, se, se_def, lo, mode, crop, fill, vmax):
    import torch
    B = imgs.shape[0]
    plan = _plan(taps, shape=imgs.shape[1:], se_values=se, se_defined=se_def, se_lo=lo, mode=mode,
                 crop=crop, img_dtype=torch.uint8, img_min=0, img_max=vmax, fill=fill, batch=B)
    plan.set_timing(True)
    d = None if defined is None else torch.from_numpy(defined.astype(np.uint8)).cuda()
    out, valid = plan.execute(torch.from_numpy(imgs).cuda(), d)
    dev = plan.read_stats()
    t = plan.get_timing(reset=True)
    return out.cpu().numpy(), valid.cpu().numpy().astype(bool), dev, t["conv_flops"]


@pytest.mark.parametrize("case", ["smooth_nonflat", "smooth_gaps_nocrop", "flat_mask", "uniform_levels"])
@pytest.mark.parametrize("mode", ["dilate", "erode"])
def test_clamp_bit_exact(case, mode):
    rng = np.random.default_rng(zlib.crc32(f"{case}/{mode}".encode()))
    defined, se_def, crop = None, None, True
    if case == "smooth_nonflat":
        imgs = np.stack([_smooth(rng, (300, 260), 64) for _ in range(2)])
        se = rng.integers(0, 16, (15, 15))
    elif case == "smooth_gaps_nocrop":
        imgs = np.stack([_smooth(rng, (200, 230), 100) for _ in range(2)])
        defined = rng.random(imgs.shape) > 0.05
        defined[:, 40:90, 50:120] = False          # a hole larger than the SE
        se = rng.integers(0, 9, (11, 7))
        se_def = rng.random(se.shape) > 0.3
        se_def[5, 3] = True
        crop = mode == "erode"                     # erosion follows erode_fft (crop only)
    elif case == "flat_mask":
        imgs = rng.integers(0, 16, (2, 400, 300)).astype(np.uint8)
        se = np.zeros((61, 61), np.int64)
        se_def = rng.random(se.shape) < 0.5
        se_def[30, 30] = True
    else:
        imgs = np.stack([np.full((150, 170), 9, np.uint8), rng.integers(0, 2, (150, 170)).astype(np.uint8)])
        se = rng.integers(0, 3, (5, 5))
    lo = tuple(-(s // 2) for s in se.shape)
    vmax = int(imgs.max())
    fill = 0 if mode == "dilate" else vmax
    out, valid, dev, fl_clamp = _run(128, imgs, defined, se, se_def, lo, mode, crop, fill, vmax)
    out0, valid0, _, fl_plain = _run(0, imgs, defined, se, se_def, lo, mode, crop, fill, vmax)
    assert dev < 0.25
    for i in range(imgs.shape[0]):
        ref, rvalid = cnaive.naive(imgs[i], None if defined is None else defined[i], se, se_def, lo,
                                   erode=(mode == "erode"), crop=crop, fill=fill)
        assert np.array_equal(valid[i], rvalid.astype(bool)), i
        assert np.array_equal(out[i].astype(np.int64), ref.astype(np.int64)), i
        assert np.array_equal(out0[i], out[i]) and np.array_equal(valid0[i], valid[i])
    if case in ("smooth_nonflat", "flat_mask"):
        assert fl_clamp < 0.8 * fl_plain, (fl_clamp, fl_plain)


def test_clamp_1d_and_wide_tiles():
    """1-D units (groups of tiles) and the 256^2 HBM tile path with the clamp."""
    import torch
    rng = np.random.default_rng(77)
    sig = np.cumsum(rng.integers(-1, 2, 20000)) % 40
    sig = sig.astype(np.uint8)[None]
    se = rng.integers(0, 6, 41)
    for mode in ("dilate", "erode"):
        fill = 0 if mode == "dilate" else 39
        out, valid, _, _ = _run(128, sig, None, se, None, (-20,), mode, True, fill, 39)
        ref, rv = cnaive.naive(sig[0], None, se, None, (-20,), erode=(mode == "erode"), fill=fill)
        assert np.array_equal(out[0].astype(np.int64), ref.astype(np.int64))
    img = _smooth(rng, (700, 650), 32)[None]
    se = rng.integers(0, 4, (101, 101))
    plan = _plan(128, shape=img.shape[1:], se_values=se, se_lo=(-50, -50), img_dtype=torch.uint8,
                 img_min=0, img_max=31, tile=256)
    out, valid = plan.execute(torch.from_numpy(img).cuda())
    ref, _ = cnaive.naive(img[0], None, se, None, (-50, -50))
    assert np.array_equal(out[0].cpu().numpy().astype(np.int64), ref.astype(np.int64))
