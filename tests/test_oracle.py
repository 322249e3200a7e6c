"""CPU: pin the oracle (and the numpy model of the kernels) to the reference.

The oracle restatements (oracle/port.py, oracle/naive.c) are checked against
  * the reference's own golden vectors (conftest.py:10-61, test_umbra.py:61-77),
  * fixtures produced by running the reference itself (tests/golden/*, made by
    tests/golden/make_golden.py), and
  * the SURVEY §8(d) input digests of the five BASELINE configs.
"""

import json

import numpy as np
import pytest

from conftest import (EXAMPLE_DILATION, EXAMPLE_IMAGE, EXAMPLE_SE, GOLDEN, RESULT_COUNT_MATRIX,
                      load_cases)
from oracle import cnaive, port
from paper_2305_03018_b200 import workloads as W


def _example_arrays():
    f = np.array(EXAMPLE_IMAGE)
    b = np.array([1, 2, 0, 0])
    bd = np.array([True, True, False, True])
    return f, b, bd


def test_worked_example_fft_and_naive():
    f, b, bd = _example_arrays()
    v, valid, lo, dev, _ = port.dilate_fft(f, None, (0,), b, bd, (-1,))
    assert v.tolist() == EXAMPLE_DILATION and valid.all() and lo == (0,)
    assert dev < 0.25
    v2, _, _ = port.dilate_naive(f, None, (0,), b, bd, (-1,))
    assert v2.tolist() == EXAMPLE_DILATION


def test_worked_example_count_matrix():
    # conftest.py:50-61 / test_umbra.py:104-112: counts over the image domain, degrees 0..9
    f, b, bd = _example_arrays()
    counts, _, _ = port.conv_full_fft(port.build_umbra(f, None, 9), port.build_umbra(b, bd, 9))
    window = counts[1:7, :10]
    expect = np.asarray(RESULT_COUNT_MATRIX)[::-1].T
    assert np.array_equal(window, expect)
    col = counts[2 - (-1)]
    assert np.flatnonzero(col).tolist() == [3, 7, 9]


def test_project_example_column():
    # test_umbra.py:73-77
    col = np.zeros((1, 10), dtype=np.int64)
    col[0, [3, 7, 9]] = 1
    v, has = port.project_with_validity(col, (2,), ((2, 2),))
    assert v.tolist() == [9] and has.all()


def test_next_fast_size_ladder():
    # fft_conv.py:61-77 and test_fft_conv.py:23-35
    for n in list(range(1, 200)) + [271, 351, 1021, 5000]:
        s = port.next_fast_size(n)
        assert s >= n
        for p in (2, 3, 5):
            while s % p == 0:
                s //= p
        assert s == 1
    assert port.next_fast_size(256 + 16 - 1) == port.next_fast_size(256 + 96 - 1)


def _grid_args(meta, arr, i):
    k = f"c{i}"
    nd = meta["nd"]
    return (arr[k + "_fv"], arr[k + "_fd"], tuple(meta["f_lo"]), arr[k + "_bv"], arr[k + "_bd"],
            tuple(meta["b_lo"]))


@pytest.mark.parametrize("which", ["port_fft", "port_naive", "c_naive"])
def test_oracle_matches_reference_cases(which):
    meta, arr = load_cases()
    for i, m in enumerate(meta):
        fv, fd, flo, bv, bd, blo = _grid_args(m, arr, i)
        k = f"c{i}"
        crop = m["crop"]
        if m["dil_error"] is None:
            if which == "port_fft":
                v, valid, lo, dev, _ = port.dilate_fft(fv, fd, flo, bv, bd, blo, crop=crop)
                assert dev < 0.25
            elif which == "port_naive":
                v, valid, lo = port.dilate_naive(fv, fd, flo, bv, bd, blo, crop=crop)
            else:
                v, valid = cnaive.naive(fv, fd, bv, bd, blo, crop=crop, fill=0, threads=2)
                lo = tuple(m["dil_lo"])
            assert np.array_equal(v, arr[k + "_dil"]), i
            assert np.array_equal(valid, arr[k + "_dilv"]), i
            assert tuple(lo) == tuple(m["dil_lo"]), i
        l = m["l"] if m["l"] is not None else m["tonal_max"]
        if m["ero_error"] is None and which == "port_fft":
            v, valid, lo, dev, _ = port.erode_fft(fv, fd, flo, bv, bd, blo, l=l)
            assert np.array_equal(v, arr[k + "_ero"]) and np.array_equal(valid, arr[k + "_erov"]), i
        if which == "port_naive":
            v, valid, lo = port.erode_naive(fv, fd, flo, bv, bd, blo, crop=crop, neutral=m["tonal_max"])
            assert np.array_equal(v, arr[k + "_eron"]) and np.array_equal(valid, arr[k + "_eronv"]), i
            assert tuple(lo) == tuple(m["eron_lo"])
        if which == "c_naive":
            v, valid = cnaive.naive(fv, fd, bv, bd, blo, erode=True, crop=crop, fill=m["tonal_max"], threads=2)
            assert np.array_equal(v, arr[k + "_eronv"] * 0 + arr[k + "_eron"]), i
            assert np.array_equal(valid, arr[k + "_eronv"]), i


def test_kernel_model_matches_reference_cases():
    """The numpy model of the CUDA index algebra reproduces the reference outputs."""
    import kernel_model as KM
    for P in (16, 32, 64, 128, 256):
        assert KM.permuted_freq_check(P)
    meta, arr = load_cases()
    checked = 0
    for i, m in enumerate(meta):
        if i % 4 or m["dil_error"] is not None:
            continue
        fv, fd, flo, bv, bd, blo = _grid_args(m, arr, i)
        if np.asarray(fv).size > 900:
            continue
        k = f"c{i}"
        v, valid, dev = KM.model_dilate(fv, fd, bv, bd, blo, mode="dilate", crop=m["crop"], fill=0)
        assert np.array_equal(v, arr[k + "_dil"]) and np.array_equal(valid, arr[k + "_dilv"]), i
        assert dev < 0.25
        l = m["l"] if m["l"] is not None else m["tonal_max"]
        v, valid, dev = KM.model_dilate(fv, fd, bv, bd, blo, mode="erode", crop=True, fill=l)
        assert np.array_equal(v, arr[k + "_ero"]) and np.array_equal(valid, arr[k + "_erov"]), i
        checked += 1
    assert checked >= 10


def test_stockham_model():
    import kernel_model as KM
    rng = np.random.default_rng(3)
    for N in (1, 2, 3, 4, 5, 8, 10, 16, 20, 40, 135, 160):
        Z = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        assert np.allclose(KM.stockham_inverse(Z, KM.radix_plan(N)), np.fft.ifft(Z) * N)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_workload_input_digests(name):
    w = W.CONFIGS[name]()
    img_d, se_d = W.EXPECTED_DIGESTS[name]
    assert W.digest(w.images[0]) == img_d
    assert W.se_digest(w.se_values, w.se_defined) == se_d


def test_workload_c5_digests():
    assert W.digest(W.c5_image(0)) == W.EXPECTED_DIGESTS["c5"][0]
    assert W.digest(W.c5_image(63)) == W.C5_IMG63_DIGEST
    assert W.se_digest(W.c5_se(), np.ones((31, 31), bool)) == W.EXPECTED_DIGESTS["c5"][1]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_small_config_golden(name):
    w = W.CONFIGS[name]()
    g = np.load(GOLDEN / f"{name}.npz")
    v, valid = cnaive.naive(w.images[0], None, w.se_values, w.se_defined, w.se_lo, crop=True, fill=0)
    assert np.array_equal(v, g["dil"]) and np.array_equal(valid, g["dilv"])
    v, valid = cnaive.naive(w.images[0], None, w.se_values, w.se_defined, w.se_lo, erode=True,
                            crop=True, fill=w.tonal_max)
    assert np.array_equal(v, g["ero"]) and np.array_equal(valid, g["erov"])


def _digest(v, valid):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(v.astype(np.int32)).tobytes()
                          + np.ascontiguousarray(valid.astype(np.uint8)).tobytes()).hexdigest()


@pytest.mark.parametrize("key", ["c3_img0", "c4_img0", "c5_img0"])
def test_c_oracle_matches_reference_digests(key):
    path = GOLDEN / "digests.json"
    if not path.exists():
        pytest.skip("digests.json not generated")
    dg = json.loads(path.read_text())
    if key not in dg:
        pytest.skip(f"{key} not in digests.json")
    name, idx = key.split("_img")
    if name == "c5":
        img, se, sd, lo, tm = W.c5_image(int(idx)), W.c5_se(), np.ones((31, 31), bool), (-15, -15), 63
    else:
        w = W.CONFIGS[name]()
        img, se, sd, lo, tm = w.images[0], w.se_values, w.se_defined, w.se_lo, w.tonal_max
    v, valid = cnaive.naive(img, None, se, sd, lo, crop=True, fill=0)
    assert _digest(v, valid) == dg[key]["dilate"]
    v, valid = cnaive.naive(img, None, se, sd, lo, erode=True, crop=True, fill=tm)
    assert _digest(v, valid) == dg[key]["erode"]


def test_clamped_unit_model_matches_oracle():
    """fm_range.cuh's clamp bound + per-unit tonal length is exact (integer model, tiny T)."""
    import kernel_model as KM
    rng = np.random.default_rng(11)
    checked = 0
    for trial in range(24):
        H, Wd = int(rng.integers(5, 40)), int(rng.integers(5, 40))
        my, mx = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        smooth = trial % 3 == 0
        if smooth:   # smooth images give strong clamps (small T_t)
            yy, xx = np.mgrid[0:H, 0:Wd]
            img = (20 + 10 * np.sin(yy / 4.0) + 10 * np.cos(xx / 5.0)).astype(np.int64)
        else:
            img = rng.integers(0, int(rng.integers(2, 60)), (H, Wd))
        fdef = rng.random((H, Wd)) > (0.3 if trial % 4 == 1 else 0.0)
        if not fdef.any():
            fdef[0, 0] = True
        se = rng.integers(0, int(rng.integers(1, 12)), (my, mx))
        sdef = rng.random((my, mx)) > (0.4 if trial % 2 else 0.0)
        sdef[0, 0] = True
        lo = (int(rng.integers(-my, 2)), int(rng.integers(-mx, 2)))
        crop = trial % 5 != 4
        cap = (4, 16, 128)[trial % 3]
        for mode in ("dilate", "erode"):
            fill = 0 if mode == "dilate" else int(img[fdef].max())
            ecrop = crop if mode == "dilate" else True
            v, valid, _ = KM.model_clamped_units(img, fdef, se, sdef, lo, mode=mode, crop=ecrop,
                                                 fill=fill, P=16, cap=cap)
            if mode == "dilate":
                rv, rvalid, _ = port.dilate_naive(img, fdef, (0, 0), se, sdef, lo, crop=crop)
            else:
                rv, rvalid, _ = port.erode_naive(img, fdef, (0, 0), se, sdef, lo, crop=True, neutral=fill)
            assert np.array_equal(valid, rvalid), (trial, mode)
            assert np.array_equal(np.where(valid, v, 0), np.where(rvalid, rv, 0)), (trial, mode)
            checked += 1
    assert checked == 48
