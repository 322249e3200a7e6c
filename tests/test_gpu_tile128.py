"""GPU: the three-pass 128x128 tile kernel (fm_tile128.cuh) against the C oracle.

Forces 128x128 tiles and walks SE widths around the window trim (the plan cuts
the valid window QX = 129 - mx to a multiple of 32 when it is 1..4 past one, so
an inverse-y warp has no output column): widths 29..32, 61..64, 93..96 trim,
others do not.  Tonal lengths above the kernel's uint8 limit (254) fall back to
the four-pass kernel, which the 8-bit cases with wide SE ranges exercise.
"""

import zlib

import numpy as np
import pytest

from oracle import cnaive

pytestmark = pytest.mark.gpu

WIDTHS = [29, 31, 32, 33, 50, 61, 64, 65, 93, 96, 100]


def _smooth(rng, shape, levels):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(rng.standard_normal(shape), float(rng.uniform(1.0, 5.0)))
    x = (x - x.min()) / max(x.max() - x.min(), 1e-9)
    return np.rint(x * (levels - 1)).astype(np.int64)


@pytest.mark.parametrize("mx", WIDTHS)
@pytest.mark.parametrize("variant", range(3))
def test_tile128_vs_oracle(mx, variant):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(zlib.crc32(f"t128/{mx}/{variant}".encode()))
    shape = (int(rng.integers(100, 400)), int(rng.integers(100, 400)))
    my = int(rng.integers(1, 100))
    levels = [16, 64, 256][variant]
    img = _smooth(rng, shape, levels) if variant != 1 else rng.integers(0, levels, shape)
    defined = rng.random(shape) > 0.2 if variant == 2 else None
    se = rng.integers(0, [16, 8, 3][variant], (my, mx))
    se_def = rng.random((my, mx)) > 0.3 if variant != 0 else None
    if se_def is not None:
        se_def[my // 2, mx // 2] = True
    se_lo = (-(my // 2) + int(rng.integers(-3, 4)), -(mx // 2) + int(rng.integers(-3, 4)))
    for mode, crop in (("dilate", True), ("erode", True), ("dilate", False)):
        fill = 0 if mode == "dilate" else levels - 1
        plan = MorphPlan(shape=shape, se_values=se, se_defined=se_def, se_lo=se_lo, mode=mode, crop=crop,
                         img_dtype=torch.uint8, img_min=0, img_max=levels - 1, fill=fill, batch=2, tile=128)
        assert plan.info["tile_x"] == 128
        imgs = np.stack([img, img[::-1, ::-1].copy()])
        defs = None if defined is None else np.stack([defined, defined[::-1, ::-1].copy()])
        d = None if defs is None else torch.from_numpy(defs.astype(np.uint8)).cuda()
        out, valid = plan.execute(torch.from_numpy(imgs.astype(np.uint8)).cuda(), d)
        assert plan.read_stats() < 0.25
        out, valid = out.cpu().numpy(), valid.cpu().numpy().astype(bool)
        for i in range(2):
            ref, rvalid = cnaive.naive(imgs[i], None if defs is None else defs[i], se, se_def, se_lo,
                                       erode=(mode == "erode"), crop=crop, fill=fill)
            assert np.array_equal(valid[i], rvalid.astype(bool)), (mode, crop, i)
            assert np.array_equal(out[i].astype(np.int64), ref.astype(np.int64)), (mode, crop, i)


@pytest.mark.parametrize("env", ["FM_TONAL_TMA=0", "FM_TRIM_QX=0", "FM_TILE3=0"])
def test_alternate_paths_bit_exact(env, monkeypatch):
    """Every plan-time A/B switch keeps the result bit-exact: per-plane bulk copies
    instead of 2-D tensor copies in the tonal kernel, the untrimmed window, the
    four-pass tile kernel."""
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    name, val = env.split("=")
    monkeypatch.setenv(name, val)
    rng = np.random.default_rng(2305)
    img = _smooth(rng, (300, 280), 64)
    se = rng.integers(0, 16, (31, 31))
    for mode in ("dilate", "erode"):
        fill = 0 if mode == "dilate" else 63
        plan = MorphPlan(shape=img.shape, se_values=se, se_lo=(-15, -15), mode=mode, img_dtype=torch.uint8,
                         img_min=0, img_max=63, fill=fill, batch=1)
        out, valid = plan.execute(torch.from_numpy(img.astype(np.uint8)[None]).cuda())
        ref, rvalid = cnaive.naive(img, None, se, None, (-15, -15), erode=(mode == "erode"), fill=fill)
        assert np.array_equal(out[0].cpu().numpy().astype(np.int64), ref.astype(np.int64)), (env, mode)
        assert np.array_equal(valid[0].cpu().numpy().astype(bool), rvalid.astype(bool)), (env, mode)


@pytest.mark.parametrize("levels,se_range", [(250, 4), (256, 3), (600, 16), (740, 30), (1000, 16)])
def test_long_tonal_axes_vs_oracle(levels, se_range):
    """Tonal lengths around the limits: 254 (uint8 tile indices), the generic tonal
    kernel's ~780 (T > 780 is refused at plan creation)."""
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(levels * 7 + se_range)
    img = rng.integers(0, levels, (200, 230))
    se = rng.integers(0, se_range, (31, 29))
    se_def = rng.random((31, 29)) > 0.2
    se_def[15, 14] = True
    for mode in ("dilate", "erode"):
        fill = 0 if mode == "dilate" else levels - 1
        try:
            plan = MorphPlan(shape=img.shape, se_values=se, se_defined=se_def, se_lo=(-15, -14), mode=mode,
                             img_dtype=torch.uint16, img_min=0, img_max=levels - 1, fill=fill, batch=1, tile=128)
        except NotImplementedError:
            assert levels + se_range > 780
            return
        out, valid = plan.execute(torch.from_numpy(img.astype(np.uint16)[None]).cuda())
        assert plan.read_stats() < 0.25
        ref, rvalid = cnaive.naive(img, None, se, se_def, (-15, -14), erode=(mode == "erode"), fill=fill)
        assert np.array_equal(out[0].cpu().numpy().astype(np.int64), ref.astype(np.int64)), (levels, mode)
        assert np.array_equal(valid[0].cpu().numpy().astype(bool), rvalid.astype(bool)), (levels, mode)
