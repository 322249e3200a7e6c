"""GPU: the functional envelope of dilate_fft / erode_fft (morphology.py:116-180 accept any
SE shape and any non-negative value range), bit-exact against the C oracle:

* long tonal axes: 10-bit and 11-bit data (tonal lengths ~1100 and ~2100: the generic
  tonal kernel with partial-warp CTAs, the four-pass tile kernel beyond 1646);
* SEs wider than one FFT tile (> 256 per axis): the plan splits the SE into blocks and
  combines the blocks' results (dilation by a union = max of the dilations, erosion =
  min, validity OR-ed) -- 400x400 and 300x300 2-D SEs, a 1000-tap 1-D SE, crop on / off,
  through the plan API and the drop-in API."""

import numpy as np
import pytest

from oracle import cnaive

pytestmark = pytest.mark.gpu


def _plan(shape, se, sd, lo, mode, vmax, crop=True, dt=None):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    dt = dt or (torch.uint8 if vmax <= 255 else torch.uint16)
    return MorphPlan(shape=shape, se_values=se, se_defined=sd, se_lo=lo, mode=mode, crop=crop, img_dtype=dt,
                     img_min=0, img_max=vmax, fill=0 if mode == "dilate" else vmax,
                     device=torch.device("cuda", 0))


def _run(img, se, sd, lo, mode, vmax, crop=True):
    import torch
    dt = torch.uint8 if vmax <= 255 else torch.uint16
    p = _plan(img.shape, se, sd, lo, mode, vmax, crop, dt)
    x = torch.from_numpy(img.astype(np.uint8 if vmax <= 255 else np.uint16)).cuda().unsqueeze(0)
    p.reset_stats()
    out, valid = p.execute(x)
    dev = p.read_stats()
    info = p.info
    p.close()
    return out[0].cpu().numpy(), valid[0].cpu().numpy().astype(bool), dev, info


@pytest.mark.parametrize("bits", [10, 11])
@pytest.mark.parametrize("mode", ["dilate", "erode"])
def test_long_tonal_axes(bits, mode):
    rng = np.random.default_rng(bits)
    top = (1 << bits) - 1
    img = rng.integers(0, top + 1, (150, 170))
    se = rng.integers(0, 21, (7, 9))
    sd = rng.random((7, 9)) < 0.8
    sd[3, 4] = True
    out, valid, dev, info = _run(img, se, sd, (-3, -4), mode, top)
    ref, refv = cnaive.naive(img, None, se, sd, (-3, -4), erode=mode == "erode", crop=True,
                             fill=0 if mode == "dilate" else top)
    assert info["tonal_len"] > top
    assert np.array_equal(out, ref) and np.array_equal(valid, refv)
    assert dev < 0.25


@pytest.mark.parametrize("mode,crop", [("dilate", True), ("erode", True), ("dilate", False)])
def test_se_400x400_split(mode, crop):
    rng = np.random.default_rng(400)
    img = rng.integers(0, 32, (520, 470))
    se = rng.integers(0, 4, (400, 400))
    sd = rng.random((400, 400)) < 0.05
    sd[200, 200] = True
    lo = (-200, -190)
    out, valid, dev, info = _run(img, se, sd, lo, mode, 31, crop)
    ref, refv = cnaive.naive(img, None, se, sd, lo, erode=mode == "erode", crop=crop,
                             fill=0 if mode == "dilate" else 31)
    assert out.shape == ref.shape
    assert np.array_equal(out, ref) and np.array_equal(valid, refv)
    assert dev < 0.25


def test_1d_se_1000_taps():
    rng = np.random.default_rng(1000)
    sig = rng.integers(0, 16, (1, 5000))
    se = rng.integers(0, 4, (1, 1000))
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    p = MorphPlan(shape=(5000,), se_values=se[0], se_lo=(-500,), mode="dilate", img_dtype=torch.uint8,
                  img_min=0, img_max=15, device=torch.device("cuda", 0))
    out, valid = p.execute(torch.from_numpy(sig[0].astype(np.uint8)).cuda().unsqueeze(0))
    ref, refv = cnaive.naive(sig[0], None, se[0], None, (-500,), erode=False, crop=True, fill=0)
    assert np.array_equal(out[0].cpu().numpy(), ref) and np.array_equal(valid[0].cpu().numpy().astype(bool), refv)


def test_dropin_api_wide_se():
    """dilate_fft / erode_fft on GridFunctions with a 300x300 gapped SE (morphology.py:116-180)."""
    import paper_2305_03018_b200 as m
    rng = np.random.default_rng(3)
    v = rng.integers(0, 64, (380, 350))
    se = rng.integers(0, 8, (300, 300))
    sd = rng.random((300, 300)) < 0.03
    sd[150, 150] = True
    f = m.GridFunction(v, tonal_max=63)
    b = m.GridFunction(se, sd, lo=(-150, -150), tonal_max=7)
    st = {}
    d, dv = m.dilate_fft(f, b, return_validity=True, stats=st)
    ref, refv = cnaive.naive(v, None, se, sd, (-150, -150), erode=False, crop=True, fill=0)
    assert np.array_equal(d.values, ref) and np.array_equal(dv, refv)
    e = m.erode_fft(f, b)
    eref, _ = cnaive.naive(v, None, se, sd, (-150, -150), erode=True, crop=True, fill=63)
    assert np.array_equal(e.values, eref)
    assert st["max_abs_deviation"] < 0.25
