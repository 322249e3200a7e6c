"""GPU: randomized engine-level parity against the C oracle (oracle/naive.c).

Every case draws an image (random or smooth, with or without gaps), an SE
(shape 1..61 per axis, random values, optional mask, lo anywhere, including
boxes that do not contain the origin), a mode, crop flag, batch and scratch
budget, runs the CUDA plan and compares values and validity bit for bit with
the direct max/min-plus oracle.  Together the cases drive every scheduling
path: clamp levels and range splits, static and dynamic plane chunks, the
pipelined and per-pixel tonal kernels, unit chunking with a tiny scratch
budget, the 256^2 HBM tile path, 1-D signals.
"""

import zlib

import numpy as np
import pytest

from oracle import cnaive

pytestmark = pytest.mark.gpu


def _smooth(rng, shape, levels):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(rng.standard_normal(shape), float(rng.uniform(1.0, 6.0)))
    x = (x - x.min()) / max(x.max() - x.min(), 1e-9)
    return np.rint(x * (levels - 1)).astype(np.int64)


def _case(seed):
    rng = np.random.default_rng(seed)
    one_d = rng.random() < 0.15
    if one_d:
        shape = (int(rng.integers(1, 30000)),)
        se_shape = (int(rng.integers(1, 200)),)
    else:
        shape = (int(rng.integers(1, 520)), int(rng.integers(1, 520)))
        se_shape = tuple(int(rng.integers(1, 62)) for _ in range(2))
    levels = int(rng.choice([2, 8, 16, 64, 256]))
    if not one_d and rng.random() < 0.5 and min(shape) > 4:
        img = _smooth(rng, shape, levels)
    else:
        img = rng.integers(0, levels, shape)
    defined = None
    if rng.random() < 0.3:
        defined = rng.random(shape) > rng.uniform(0.0, 0.5)
        if not defined.any():
            defined.flat[0] = True
    se = rng.integers(0, int(rng.choice([1, 2, 4, 16, 40])), se_shape)
    se_def = None
    if rng.random() < 0.4:
        se_def = rng.random(se_shape) > 0.5
        se_def.flat[int(rng.integers(0, se_def.size))] = True
    se_lo = tuple(int(rng.integers(-s - 3, 4)) for s in se_shape)
    mode = "erode" if rng.random() < 0.4 else "dilate"
    crop = rng.random() < 0.7
    batch = int(rng.integers(1, 4))
    scratch = int(rng.choice([0, 0, 1]))   # 1 byte: one unit per launch
    tile = 0
    if not one_d and rng.random() < 0.15:
        tile = 256
    dtype = str(rng.choice(["uint8", "uint8", "uint16", "int32"]))
    offset = 0
    if dtype == "uint16":
        offset = int(rng.integers(0, 60000))
    elif dtype == "int32":
        offset = int(rng.integers(-(1 << 28), 1 << 28))   # the C oracle is exact below 2^29
    return dict(shape=shape, img=img, defined=defined, se=se, se_def=se_def, se_lo=se_lo, mode=mode, crop=crop,
                batch=batch, scratch=scratch, tile=tile, levels=levels, dtype=dtype, offset=offset)


@pytest.mark.parametrize("seed", list(range(160)))
def test_fuzz_engine_vs_oracle(seed):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    c = _case(zlib.crc32(f"fuzz/{seed}".encode()))
    vals = c["img"] if c["defined"] is None else c["img"][c["defined"]]
    off = c["offset"]
    img_min, img_max = off, off + c["levels"] - 1
    fill = 0 if c["mode"] == "dilate" else img_max
    tdt = {"uint8": torch.uint8, "uint16": torch.uint16, "int32": torch.int32}[c["dtype"]]
    npdt = {"uint8": np.uint8, "uint16": np.uint16, "int32": np.int32}[c["dtype"]]
    imgs = np.stack([np.roll(c["img"], i, axis=-1) for i in range(c["batch"])]) + off
    defs = None if c["defined"] is None else np.stack([np.roll(c["defined"], i, axis=-1) for i in range(c["batch"])])
    try:
        plan = MorphPlan(shape=c["shape"], se_values=c["se"], se_defined=c["se_def"], se_lo=c["se_lo"], mode=c["mode"],
                         crop=c["crop"], img_dtype=tdt, img_min=img_min, img_max=img_max, fill=fill,
                         batch=c["batch"], scratch_bytes=c["scratch"], tile=c["tile"])
    except NotImplementedError:
        pytest.skip("configuration outside the FFT path's limits")
    d = None if defs is None else torch.from_numpy(defs.astype(np.uint8)).cuda()
    out, valid = plan.execute(torch.from_numpy(imgs.astype(npdt)).cuda(), d)
    dev = plan.read_stats()
    assert dev < 0.25
    out = out.cpu().numpy()
    valid = valid.cpu().numpy().astype(bool)
    for i in range(c["batch"]):
        ref, rvalid = cnaive.naive(imgs[i], None if defs is None else defs[i], c["se"], c["se_def"], c["se_lo"],
                                   erode=(c["mode"] == "erode"), crop=c["crop"], fill=fill)
        assert np.array_equal(valid[i], rvalid.astype(bool)), (seed, i)
        assert np.array_equal(out[i].astype(np.int64), ref.astype(np.int64)), (seed, i)
    assert vals.size > 0


@pytest.mark.parametrize("offset", [-2_000_000_000, 1_500_000_000, 2_147_483_000])
def test_large_int32_values_vs_int64_oracle(offset):
    """int32 images near the type's limits (the int64 numpy oracle, as the reference)."""
    import torch
    from oracle import port
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(abs(offset) % 1000)
    img = _smooth(rng, (150, 170), 40) + offset - (40 if offset > 0 else 0)
    se = rng.integers(0, 7, (9, 11))
    lo_v, hi_v = int(img.min()), int(img.max())
    for mode in ("dilate", "erode"):
        fill = 0 if mode == "dilate" else hi_v
        hi_out = hi_v + int(se.max()) if mode == "dilate" else hi_v
        if hi_out >= 2**31 or lo_v - int(se.max()) < -2**31:
            continue
        plan = MorphPlan(shape=img.shape, se_values=se, se_lo=(-4, -5), mode=mode, img_dtype=torch.int32,
                         img_min=lo_v, img_max=hi_v, fill=fill)
        out, valid = plan.execute(torch.from_numpy(img.astype(np.int32)).cuda())
        if mode == "dilate":
            ref, rvalid, _ = port.dilate_naive(img, None, (0, 0), se, None, (-4, -5))
        else:
            ref, rvalid, _ = port.erode_naive(img, None, (0, 0), se, None, (-4, -5), neutral=fill)
        assert np.array_equal(out[0].cpu().numpy().astype(np.int64), ref)
        assert np.array_equal(valid[0].cpu().numpy().astype(bool), rvalid)


def test_stage_reuse_race_regression():
    """Fuzz case 124 (int32, gaps, 58x33 SE, T = 270) run repeatedly over a device
    heap pre-filled with garbage: it caught a write-after-read race between the
    consumers' generic-proxy reads of a pipeline stage and the producer's next
    async-proxy (TMA) copy into it (fixed by fence.proxy.async before the
    release); ~7% of runs failed without the fence."""
    import torch
    for r in range(15):
        junk = torch.full((int(1e9) // 4,), float(r) + 0.5, dtype=torch.float32, device="cuda")
        del junk
        test_fuzz_engine_vs_oracle(124)


def _wide_case(seed):
    """Round-2 envelope: SE value ranges up to 255 (wider than the short ladder entries),
    8..11-bit data, every tile engine forced, SEs wider than one tile (split and combined),
    output windows (crop = 2) and device-dispatched small launches."""
    rng = np.random.default_rng(seed)
    shape = (int(rng.integers(3, 300)), int(rng.integers(3, 300)))
    big_se = rng.random() < 0.15
    se_shape = tuple(int(rng.integers(100, 330)) if big_se else int(rng.integers(1, 40)) for _ in range(2))
    levels = int(rng.choice([16, 256, 1024, 2048]))
    img = rng.integers(0, levels, shape)
    se_top = int(rng.choice([1, 64, 200, 255]))
    se = rng.integers(0, se_top + 1, se_shape)
    se_def = rng.random(se_shape) > (0.97 if big_se else 0.4)
    se_def.flat[int(rng.integers(0, se_def.size))] = True
    se_lo = tuple(int(-(s // 2) + rng.integers(-3, 4)) for s in se_shape)
    mode = "erode" if rng.random() < 0.4 else "dilate"
    window = None
    if rng.random() < 0.25:
        window = ((int(rng.integers(-5, shape[0])), int(rng.integers(-5, shape[1]))),
                  (int(rng.integers(1, shape[0] + 5)), int(rng.integers(1, shape[1] + 5))))
    tile = 0 if big_se else int(rng.choice([0, 0, 16, 32, 64, 128, 256]))
    if tile and max(se_shape) > tile:
        tile = 0
    return dict(shape=shape, img=img, se=se, se_def=se_def, se_lo=se_lo, mode=mode, window=window, tile=tile,
                levels=levels)


@pytest.mark.parametrize("seed", list(range(60)))
def test_fuzz_wide_ranges_vs_oracle(seed):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    c = _wide_case(zlib.crc32(f"fuzz-wide/{seed}".encode()))
    vmax = c["levels"] - 1
    fill = 0 if c["mode"] == "dilate" else vmax
    dt, npdt = (torch.uint8, np.uint8) if vmax <= 255 else (torch.uint16, np.uint16)
    try:
        plan = MorphPlan(shape=c["shape"], se_values=c["se"], se_defined=c["se_def"], se_lo=c["se_lo"],
                         mode=c["mode"], crop=True, img_dtype=dt, img_min=0, img_max=vmax, fill=fill,
                         tile=c["tile"], window=c["window"])
    except NotImplementedError:
        pytest.skip("configuration outside the FFT path's limits")
    out, valid = plan.execute(torch.from_numpy(c["img"].astype(npdt)).cuda().unsqueeze(0))
    assert plan.read_stats() < 0.25
    out, valid = out[0].cpu().numpy(), valid[0].cpu().numpy().astype(bool)
    erode = c["mode"] == "erode"
    if c["window"] is None:
        ref, rvalid = cnaive.naive(c["img"], None, c["se"], c["se_def"], c["se_lo"], erode=erode, crop=True, fill=fill)
    else:
        full, fvalid = cnaive.naive(c["img"], None, c["se"], c["se_def"], c["se_lo"], erode=erode, crop=False,
                                    fill=fill)
        my, mx = c["se"].shape
        lo = c["se_lo"]
        off = (-(lo[0] + my - 1), -(lo[1] + mx - 1)) if erode else lo
        (wy, wx), (wh, ww) = c["window"]
        ref = np.full((wh, ww), fill, np.int64)
        rvalid = np.zeros((wh, ww), bool)
        ys = np.arange(wh) + wy - off[0]
        xs = np.arange(ww) + wx - off[1]
        oky = (ys >= 0) & (ys < full.shape[0])
        okx = (xs >= 0) & (xs < full.shape[1])
        ref[np.ix_(oky, okx)] = full[np.ix_(ys[oky], xs[okx])]
        rvalid[np.ix_(oky, okx)] = fvalid[np.ix_(ys[oky], xs[okx])]
    assert np.array_equal(valid, rvalid.astype(bool)), seed
    assert np.array_equal(out.astype(np.int64), ref.astype(np.int64)), seed
