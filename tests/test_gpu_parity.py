"""GPU parity: the sm_100a path against the reference's golden outputs and the oracle.

Mirrors the reference's own assertions (test_morphology.py:100-312,
test_acceptance.py criteria 1/2/7) through the drop-in API, then checks the
BASELINE configs: c1/c2 bit-exact against full reference outputs, c3/c4/c5
bit-exact against sha256 digests of the reference's exact outputs.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import (EXAMPLE_DILATION, GOLDEN, flat_se, identity_se, load_cases, random_grid)
from oracle import cnaive, port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2305_03018_b200 import build
    build.build()


def M():
    import paper_2305_03018_b200 as m
    return m


def G(*a, **k):
    return M().GridFunction(*a, **k)


def _naive_ref(f, b, crop=True):
    v, valid, lo = port.dilate_naive(f.values, f.defined, f.lo, b.values, b.defined, b.lo, crop=crop)
    return v, valid, lo


def _erode_ref(f, b, crop=True):
    v, valid, lo = port.erode_naive(f.values, f.defined, f.lo, b.values, b.defined, b.lo, crop=crop,
                                    neutral=f.tonal_max)
    return v, valid, lo


# ------------------------------------------------------------------ reference test-suite semantics
class TestDilateFft:
    def test_worked_example(self, example_image, example_se):
        assert M().dilate_fft(example_image, example_se).to_list() == EXAMPLE_DILATION

    def test_constant_zero(self):
        z = G(np.zeros((5, 5), dtype=np.int64), tonal_max=1)
        out = M().dilate_fft(z, flat_se(3, ndim=2))
        assert not out.values.any()

    def test_matches_naive_randomized(self):
        rng = np.random.default_rng(53)
        for _ in range(20):
            f = random_grid(rng, (11, 9), 15, gap_p=0.2)
            b = random_grid(rng, (4, 3), 7, gap_p=0.3, lo=(-2, -1))
            if not b.defined.any():
                continue
            fast, valid = M().dilate_fft(f, b, return_validity=True)
            v, vv, lo = _naive_ref(f, b)
            assert np.array_equal(fast.values, v) and np.array_equal(valid, vv) and fast.lo == lo

    def test_matches_naive_uncropped(self):
        rng = np.random.default_rng(59)
        f = random_grid(rng, (7,), 9)
        b = random_grid(rng, (3,), 4, lo=(1,))
        fast = M().dilate_fft(f, b, crop=False)
        v, _, lo = _naive_ref(f, b, crop=False)
        assert fast.lo == lo and np.array_equal(fast.values, v)

    def test_stats_reported(self, example_image, example_se):
        stats = {}
        M().dilate_fft(example_image, example_se, stats=stats)
        assert 0 <= stats["max_abs_deviation"] < 0.25
        assert "padded_shape" in stats

    def test_negative_input_rejected(self):
        f = G(np.array([-1, 2]), tonal_max=3, signed=True)
        with pytest.raises(ValueError):
            M().dilate_fft(f, identity_se())

    def test_empty_intersection_quirk(self):
        # reference raises TypeError here; naive returns zeros/invalid
        f = G(np.array([1, 2]), tonal_max=3)
        b = G(np.array([0]), lo=(5,), tonal_max=1)
        with pytest.raises(TypeError):
            M().dilate_fft(f, b)
        out, valid = M().dilate_naive(f, b, return_validity=True)
        assert not valid.any() and not out.values.any()

    def test_se_far_from_origin_uncropped(self):
        f = G(np.array([1, 2, 3]), tonal_max=3)
        b = G(np.array([2, 0]), lo=(7,), tonal_max=2)
        fast, valid = M().dilate_fft(f, b, crop=False, return_validity=True)
        v, vv, lo = _naive_ref(f, b, crop=False)
        assert fast.lo == lo == (7,) and np.array_equal(fast.values, v) and np.array_equal(valid, vv)


class TestErodeFft:
    def test_interior_worked_example(self, example_image):
        fast = M().erode_fft(example_image, flat_se(3), l=7)
        assert fast.to_list()[1:5] == [0, 0, 2, 2]

    def test_identity_se(self, example_image):
        assert M().erode_fft(example_image, identity_se()) == example_image

    def test_matches_naive_everywhere(self):
        rng = np.random.default_rng(67)
        for _ in range(20):
            f = random_grid(rng, (10, 8), 15)
            b = random_grid(rng, (3, 3), 6, gap_p=0.2, lo=(-1, -1))
            got, valid = M().erode_fft(f, b, return_validity=True)
            v, vv, lo = _erode_ref(f, b)
            assert np.array_equal(got.values, v) and np.array_equal(valid, vv)

    def test_l_below_max_rejected(self, example_image):
        with pytest.raises(ValueError):
            M().erode_fft(example_image, flat_se(3), l=5)

    def test_can_go_negative(self):
        f = G(np.array([0, 0, 0]), tonal_max=5)
        b = G(np.array([3]), lo=(0,), tonal_max=3)
        assert M().erode_fft(f, b).to_list() == [-3, -3, -3]
        assert M().erode_naive(f, b).to_list() == [-3, -3, -3]


class TestNaiveGpu:
    def test_worked_example(self, example_image, example_se):
        assert M().dilate_naive(example_image, example_se).to_list() == EXAMPLE_DILATION

    def test_flat(self, example_image):
        assert M().dilate_naive(example_image, flat_se(3)).to_list() == [3, 7, 7, 7, 7, 7]
        assert M().erode_naive(example_image, flat_se(3)).to_list() == [0, 0, 0, 2, 2, 2]

    def test_random_vs_oracle(self):
        rng = np.random.default_rng(11)
        for t in range(30):
            nd = 1 + t % 2
            sh = tuple(int(x) for x in rng.integers(1, 40, nd))
            ms = tuple(int(x) for x in rng.integers(1, 9, nd))
            f = random_grid(rng, sh, 20, gap_p=0.2)
            b = random_grid(rng, ms, 5, gap_p=0.3, lo=tuple(int(x) for x in rng.integers(-6, 4, nd)))
            for crop in (True, False):
                g, gv = M().dilate_naive(f, b, crop=crop, return_validity=True)
                v, vv, lo = _naive_ref(f, b, crop=crop)
                assert np.array_equal(g.values, v) and np.array_equal(gv, vv) and g.lo == lo
                g, gv = M().erode_naive(f, b, crop=crop, return_validity=True)
                v, vv, lo = _erode_ref(f, b, crop=crop)
                assert np.array_equal(g.values, v) and np.array_equal(gv, vv) and g.lo == lo


class TestCompound:
    def test_opening_identity_se(self, example_image):
        for method in M().MorphMethod:
            assert M().opening(example_image, identity_se(), method) == example_image

    def test_gradient_constant(self):
        c = G(np.full((6, 6), 4), tonal_max=7)
        for method in M().MorphMethod:
            assert not M().beucher_gradient(c, flat_se(3, ndim=2), method).values.any()

    def test_open_close_methods_agree(self):
        rng = np.random.default_rng(71)
        f = random_grid(rng, (16, 16), 15)
        b = flat_se(5, ndim=2)
        for op in (M().opening, M().closing, M().beucher_gradient):
            a = op(f, b, M().MorphMethod.NAIVE)
            c = op(f, b, M().MorphMethod.FFT_UMBRA)
            assert np.array_equal(a.values, c.values), op.__name__

    def test_nonflat_compound_agree(self):
        # erosion intermediate goes negative; exercises the value-shift path
        rng = np.random.default_rng(73)
        f = random_grid(rng, (12, 12), 7)
        b = G(rng.integers(3, 8, (3, 3)), lo=(-1, -1), tonal_max=7)
        for op in (M().opening, M().closing, M().beucher_gradient):
            a = op(f, b, M().MorphMethod.NAIVE)
            c = op(f, b, M().MorphMethod.FFT_UMBRA)
            assert np.array_equal(a.values, c.values), op.__name__

    def test_dispatch(self, example_image, example_se):
        assert M().dilate(example_image, example_se, "fft").to_list() == EXAMPLE_DILATION
        assert M().erode(example_image, flat_se(3), "naive") == M().erode(example_image, flat_se(3), "fft")


# ------------------------------------------------------------------ reference-generated fixtures
def test_reference_cases_bit_exact():
    """120 randomized cases (gaps, any SE lo, crop on/off, 1-D and 2-D, explicit l)
    against outputs of the reference itself (tests/golden/make_golden.py)."""
    meta, arr = load_cases()
    worst = 0.0
    for i, m in enumerate(meta):
        k = f"c{i}"
        f = G(arr[k + "_fv"], arr[k + "_fd"], lo=tuple(m["f_lo"]), tonal_max=m["tonal_max"])
        b = G(arr[k + "_bv"], arr[k + "_bd"], lo=tuple(m["b_lo"]), tonal_max=m["b_tonal_max"])
        if m["dil_error"] is None:
            st = {}
            d, dv = M().dilate_fft(f, b, crop=m["crop"], return_validity=True, stats=st)
            assert np.array_equal(d.values, arr[k + "_dil"]), i
            assert np.array_equal(dv, arr[k + "_dilv"]), i
            assert d.lo == tuple(m["dil_lo"]) and d.tonal_max == m["dil_tonal_max"], i
            worst = max(worst, st["max_abs_deviation"])
        if m["ero_error"] is None:
            e, ev = M().erode_fft(f, b, l=m["l"], return_validity=True)
            assert np.array_equal(e.values, arr[k + "_ero"]) and np.array_equal(ev, arr[k + "_erov"]), i
            assert e.lo == tuple(m["ero_lo"]) and e.tonal_max == m["ero_tonal_max"], i
        en, env = M().erode_naive(f, b, crop=m["crop"], return_validity=True)
        assert np.array_equal(en.values, arr[k + "_eron"]) and np.array_equal(env, arr[k + "_eronv"]), i
    assert worst < 0.25
    print(f"\nreference cases: worst pre-rounding deviation {worst:.3e} (margin {0.5 / max(worst, 1e-30):.0f}x to 0.5)")


# ------------------------------------------------------------------ BASELINE configs
def _digest(v, valid):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(v).astype(np.int32)).tobytes()
                          + np.ascontiguousarray(np.asarray(valid).astype(np.uint8)).tobytes()).hexdigest()


def _plan_run(w, mode, imgs=None, **kw):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    imgs = w.images if imgs is None else imgs
    dt = torch.int32 if imgs.dtype == np.int32 else torch.uint8
    plan = MorphPlan(shape=imgs.shape[1:], se_values=w.se_values, se_defined=w.se_defined, se_lo=w.se_lo,
                     mode=mode, crop=True, img_dtype=dt, img_min=0, img_max=w.tonal_max,
                     fill=0 if mode == "dilate" else w.tonal_max, batch=imgs.shape[0], **kw)
    x = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    plan.reset_stats()
    out, valid = plan.execute(x)
    dev = plan.read_stats()
    return out.cpu().numpy(), valid.cpu().numpy(), dev, plan


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_small_configs_vs_reference_outputs(name):
    from paper_2305_03018_b200 import workloads as W
    w = W.CONFIGS[name]()
    g = np.load(GOLDEN / f"{name}.npz")
    # drop-in API (GridFunction in, GridFunction out)
    f = G(w.images[0].astype(np.int64), tonal_max=w.tonal_max)
    b = G(w.se_values, w.se_defined, lo=w.se_lo, tonal_max=w.se_tonal_max)
    st = {}
    d, dv = M().dilate_fft(f, b, return_validity=True, stats=st)
    assert np.array_equal(d.values, g["dil"]) and np.array_equal(dv, g["dilv"])
    e, ev = M().erode_fft(f, b, return_validity=True)
    assert np.array_equal(e.values, g["ero"]) and np.array_equal(ev, g["erov"])
    # batched plan API
    v, valid, dev, _ = _plan_run(w, "dilate")
    assert np.array_equal(v[0], g["dil"]) and np.array_equal(valid[0].astype(bool), g["dilv"])
    assert dev < 0.25
    print(f"\n{name}: max pre-rounding deviation {st['max_abs_deviation']:.3e}")


def _digests():
    return json.loads((GOLDEN / "digests.json").read_text())


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_large_configs_vs_reference_digests(name):
    from paper_2305_03018_b200 import workloads as W
    dg = _digests()[f"{name}_img0"]
    w = W.CONFIGS[name]()
    v, valid, dev, plan = _plan_run(w, "dilate")
    assert _digest(v[0], valid[0]) == dg["dilate"]
    v, valid, dev2, _ = _plan_run(w, "erode")
    assert _digest(v[0], valid[0]) == dg["erode"]
    print(f"\n{name}: T={plan.info['tonal_len']} tile={plan.info['tile_x']} dev={max(dev, dev2):.3e}")


def test_c5_vs_reference_digests():
    from paper_2305_03018_b200 import workloads as W
    dg = _digests()
    idx = [0, 1, 63]
    imgs = np.stack([W.c5_image(i) for i in idx])
    w = W.Workload("c5", imgs, W.c5_se(), np.ones((31, 31), bool), (-15, -15), 63, 6)
    v, valid, dev, plan = _plan_run(w, "dilate")
    e, ev, dev2, _ = _plan_run(w, "erode")
    for j, i in enumerate(idx):
        assert _digest(v[j], valid[j]) == dg[f"c5_img{i}"]["dilate"], i
        assert _digest(e[j], ev[j]) == dg[f"c5_img{i}"]["erode"], i
    print(f"\nc5: T={plan.info['tonal_len']} tile={plan.info['tile_x']} dev={max(dev, dev2):.3e}")


# ------------------------------------------------------------------ plan-level invariances / edges
def test_tile_and_tonal_length_invariance():
    rng = np.random.default_rng(5)
    from paper_2305_03018_b200 import workloads as W
    img = rng.integers(0, 32, (1, 150, 170)).astype(np.uint8)
    se = rng.integers(0, 5, (9, 13))
    sd = rng.random((9, 13)) > 0.3
    sd[4, 6] = True
    w = W.Workload("x", img, se, sd, (-4, -2), 31, 5)
    ref, refv = cnaive.naive(img[0], None, se, sd, (-4, -2), crop=True, fill=0)
    for tile in (16, 32, 64, 128, 256):
        v, valid, dev, plan = _plan_run(w, "dilate", tile=tile)
        assert plan.info["tile_x"] == tile
        assert np.array_equal(v[0], ref) and np.array_equal(valid[0].astype(bool), refv), tile
    for T in (36, 40, 64, 80, 162, 270, 400):   # register, shared-memory and generic tonal kernels
        v, valid, dev, plan = _plan_run(w, "dilate", tonal_len=T)
        assert plan.info["tonal_len"] == T
        assert np.array_equal(v[0], ref), T


COOP_NS = [45, 48, 50, 54, 60, 64, 72, 75, 80, 81, 90, 96, 100, 108, 120, 125, 128, 135, 144, 150, 160]


@pytest.mark.parametrize("N", COOP_NS + [40, 162, 180])
def test_long_tonal_axes_every_ladder_entry(N, monkeypatch):
    """Every tonal length 2N served by the several-threads-per-pixel kernel
    (fm_tonal_coop.cuh, 40 < N <= 160) and its neighbours (pipelined register kernel,
    generic kernel): uniform data whose spread needs exactly that ladder entry (the clamp
    bound is switched off so no tile gets a shorter one), dilation and erosion, an SE with gaps."""
    from paper_2305_03018_b200 import workloads as W
    monkeypatch.setenv("FM_RANGE_TAPS", "0")
    rng = np.random.default_rng(1000 + N)
    vmax = 2 * N - 1 - 4
    img = rng.integers(0, vmax + 1, (1, 131, 157)).astype(np.int32)
    img[0, 0, 0], img[0, 5, 7], img[0, 100, 120] = 0, vmax, vmax
    img[0, 70, 80] = 0
    se = rng.integers(0, 5, (5, 7))
    se[0, 0], se[4, 6] = 0, 4
    sd = rng.random((5, 7)) > 0.2
    sd[0, 0] = sd[4, 6] = sd[2, 3] = True
    bits = int(vmax).bit_length()
    w = W.Workload("x", img, se, sd, (-2, -3), vmax, bits)
    for mode in ("dilate", "erode"):
        v, valid, dev, plan = _plan_run(w, mode)
        assert plan.info["tonal_len"] >= 2 * N
        ref, refv = cnaive.naive(img[0].astype(np.int64), None, se, sd, (-2, -3), erode=(mode == "erode"), crop=True,
                                 fill=0 if mode == "dilate" else vmax)
        assert np.array_equal(v[0], ref) and np.array_equal(valid[0].astype(bool), refv), (N, mode)
        assert dev < 0.25


def test_long_tonal_axes_mixed_entries_one_launch(monkeypatch):
    """Tiles of one image with very different spreads: many ladder entries of the
    several-threads-per-pixel kernel in flight at once (one launch each, side by side on the
    tonal streams) beside the device-dispatched launch of the short entries."""
    from paper_2305_03018_b200 import workloads as W
    monkeypatch.setenv("FM_RANGE_TAPS", "0")
    rng = np.random.default_rng(77)
    H = Wd = 520
    img = np.zeros((1, H, Wd), np.int32)
    spreads = [20, 60, 88, 100, 118, 140, 160, 200, 236, 250, 280, 300]
    k = 0
    for by in range(0, H, 130):
        for bx in range(0, Wd, 130):
            sp = spreads[k % len(spreads)]
            k += 1
            img[0, by:by + 130, bx:bx + 130] = rng.integers(0, sp + 1, (min(130, H - by), min(130, Wd - bx)))
    se = rng.integers(0, 4, (9, 9))
    se[0, 0], se[8, 8] = 0, 3
    w = W.Workload("x", img, se, np.ones((9, 9), bool), (-4, -4), 300, 9)
    for mode in ("dilate", "erode"):
        v, valid, dev, plan = _plan_run(w, mode, tile=128)
        assert plan.info["tile_x"] == 128
        ref, refv = cnaive.naive(img[0], None, se, None, (-4, -4), erode=(mode == "erode"), crop=True,
                                 fill=0 if mode == "dilate" else 300)
        assert np.array_equal(v[0], ref) and np.array_equal(valid[0].astype(bool), refv), mode
        assert dev < 0.25


@pytest.mark.parametrize("tile", [16, 32, 64, 128, 256])
def test_se_value_range_wider_than_short_ladder_entries(tile):
    """8-bit data with an SE whose own value range (up to 230) exceeds the shortest ladder
    entries: their (never used) SE spectra must stay in bounds for every tile engine
    (regression: the four-pass kernels indexed a per-plane table of T + 1 entries with
    unreduced SE values)."""
    from paper_2305_03018_b200 import workloads as W
    rng = np.random.default_rng(230 + tile)
    edge = max(tile - 2, 12)
    img = rng.integers(0, 256, (1, edge, edge + 5)).astype(np.uint8)
    se = rng.integers(0, 231, (3, 3))
    se[0, 0], se[2, 2] = 0, 230
    w = W.Workload("x", img, se, np.ones((3, 3), bool), (-1, -1), 255, 8)
    for mode in ("dilate", "erode"):
        v, valid, dev, plan = _plan_run(w, mode, tile=tile)
        ref, refv = cnaive.naive(img[0], None, se, None, (-1, -1), erode=(mode == "erode"), crop=True,
                                 fill=0 if mode == "dilate" else 255)
        assert np.array_equal(v[0], ref) and np.array_equal(valid[0].astype(bool), refv), (tile, mode)


def test_wide_se_big_tiles():
    """SEs wider than the 128 SMEM tile run on 256x256 tiles through HBM (fm_bigtile.cuh)."""
    from paper_2305_03018_b200 import workloads as W
    rng = np.random.default_rng(77)
    img = rng.integers(0, 10, (2, 300, 283)).astype(np.uint8)
    se = rng.integers(0, 3, (150, 141))
    sd = rng.random((150, 141)) > 0.6
    sd[75, 70] = True
    w = W.Workload("x", img, se, sd, (-75, -60), 9, 4)
    for mode in ("dilate", "erode"):
        v, valid, dev, plan = _plan_run(w, mode)
        assert plan.info["tile_x"] == 256
        for i in range(2):
            ref, refv = cnaive.naive(img[i], None, se, sd, (-75, -60), erode=(mode == "erode"), crop=True,
                                     fill=0 if mode == "dilate" else 9)
            assert np.array_equal(v[i], ref) and np.array_equal(valid[i].astype(bool), refv), (mode, i)
    # drop-in API, gaps in the image, uncropped
    f = random_grid(rng, (140, 170), 12, gap_p=0.1)
    b = random_grid(rng, (131, 9), 3, gap_p=0.5, lo=(-70, -4))
    d, dv = M().dilate_fft(f, b, crop=False, return_validity=True)
    rv, rvv, lo = _naive_ref(f, b, crop=False)
    assert d.lo == lo and np.array_equal(d.values, rv) and np.array_equal(dv, rvv)


def test_batch_chunking_and_host_path():
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(9)
    imgs = rng.integers(0, 16, (5, 70, 90)).astype(np.uint8)
    se = rng.integers(0, 4, (7, 7))
    plan = MorphPlan(shape=(70, 90), se_values=se, se_lo=(-3, -3), img_dtype=torch.uint8, img_min=0,
                     img_max=15, batch=5, scratch_bytes=1)   # forces one image per launch
    assert plan.info["images_per_launch"] == 1
    assert plan.info["scratch_bytes"] < 70 * 90 * 8 * 64   # one tile's planes per launch (unit chunking)
    out, valid = plan.execute(torch.from_numpy(imgs).cuda())
    host_out, host_valid = plan.execute_host(imgs)
    for i in range(5):
        ref, _ = cnaive.naive(imgs[i], None, se, None, (-3, -3))
        assert np.array_equal(out[i].cpu().numpy(), ref)
        assert np.array_equal(host_out[i].numpy(), ref)


def test_value_range_error_detected():
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    plan = MorphPlan(shape=(32, 32), se_values=np.zeros((3, 3)), se_lo=(-1, -1), img_dtype=torch.uint8,
                     img_min=0, img_max=7)
    x = torch.full((1, 32, 32), 9, dtype=torch.uint8, device="cuda")
    plan.reset_stats()
    plan.execute(x)
    with pytest.raises(ValueError):
        plan.read_stats()


def test_gaps_and_offsets_large_1d():
    rng = np.random.default_rng(21)
    n = 20000
    f = random_grid(rng, (n,), 40, gap_p=0.1)
    b = random_grid(rng, (200,), 9, gap_p=0.2, lo=(-37,))
    for crop in (True, False):
        d, dv = M().dilate_fft(f, b, crop=crop, return_validity=True)
        v, vv, lo = _naive_ref(f, b, crop=crop)
        assert np.array_equal(d.values, v) and np.array_equal(dv, vv) and d.lo == lo
    e, ev = M().erode_fft(f, b, return_validity=True)
    v, vv, _ = _erode_ref(f, b)
    assert np.array_equal(e.values, v) and np.array_equal(ev, vv)


def test_reference_grid_interop_roundtrip():
    # a reference-shaped object (duck type) is accepted and compares equal
    class Foreign:
        def __init__(self, g):
            self.values, self.defined, self.lo, self.tonal_max, self.signed = g.values, g.defined, g.lo, g.tonal_max, g.signed
    rng = np.random.default_rng(2)
    f = random_grid(rng, (20, 20), 15)
    b = flat_se(3, ndim=2)
    d = M().dilate_fft(Foreign(f), Foreign(b))
    assert d == Foreign(M().dilate_naive(f, b))


def test_launch_counter_advances():
    from paper_2305_03018_b200 import _lib
    before = _lib.kernel_launches()
    M().dilate_fft(G(np.arange(10) % 4, tonal_max=3), flat_se(3))
    assert _lib.kernel_launches() >= before + 2


@pytest.mark.parametrize("seed", range(8))
def test_flat_wide_se_regime_fuzz(seed):
    """The c4 regime in small: few-bit images, wide flat SEs with random masks, batches, image gaps --
    256x256 tiles with paired Nyquist planes, the compact job list, the short-axis tonal kernel and
    the range kernel's int8 windows / flat-tap walk, against the C oracle."""
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(4000 + seed)
    bits = int(rng.integers(1, 6))
    vmax = (1 << bits) - 1
    H, Wd = int(rng.integers(260, 560)), int(rng.integers(260, 560))
    if seed % 2 == 0:
        Wd = (Wd + 15) & ~15                      # 16-byte aligned rows: the chunk-aligned staging paths
    my, mx = int(rng.integers(65, 150)), int(rng.integers(65, 150))
    batch = int(rng.integers(1, 4))
    img = rng.integers(0, vmax + 1, (batch, H, Wd)).astype(np.uint8)
    sd = rng.random((my, mx)) < rng.uniform(0.2, 0.9)
    sd[my // 2, mx // 2] = True
    se = np.zeros((my, mx), np.int64)
    lo = (-int(rng.integers(0, my)), -int(rng.integers(0, mx)))
    gaps = seed % 3 == 2
    defined = (rng.random((batch, H, Wd)) > 0.05) if gaps else None
    for mode in ("dilate", "erode"):
        fill = 0 if mode == "dilate" else vmax
        plan = MorphPlan(shape=(H, Wd), se_values=se, se_defined=sd, se_lo=lo, mode=mode, crop=True,
                         img_dtype=torch.uint8, img_min=0, img_max=vmax, fill=fill, batch=batch)
        assert plan.info["tile_x"] == 256
        x = torch.from_numpy(img).cuda()
        dm = None if defined is None else torch.from_numpy(defined.astype(np.uint8)).cuda()
        plan.reset_stats()
        out, valid = plan.execute(x, dm)
        assert plan.read_stats() < 0.25
        for i in range(batch):
            ref, refv = cnaive.naive(img[i], None if defined is None else defined[i], se, sd, lo,
                                     erode=(mode == "erode"), crop=True, fill=fill)
            assert np.array_equal(out[i].cpu().numpy(), ref), (seed, mode, i)
            assert np.array_equal(valid[i].cpu().numpy().astype(bool), refv), (seed, mode, i)
