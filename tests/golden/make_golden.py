"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed; nothing reads /root/reference at test time):
  cases.npz      small randomized cases (gaps, arbitrary SE lo, crop on/off,
                 1-D and 2-D, erosion with explicit l) with the reference's
                 dilate_fft / erode_fft / dilate_naive / erode_naive outputs and
                 stats["max_abs_deviation"]
  c1.npz, c2.npz full reference outputs at BASELINE configs c1 and c2
  digests.json   sha256 of the reference's exact outputs at c3, c4 and c5
                 (images 0, 1, 63): dilate_naive / erode_naive, which the
                 reference's own tests prove equal to dilate_fft / erode_fft
                 (test_morphology.py:179-189, test_acceptance.py:69-98)
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from fftmorph.morphology import (dilate_fft, dilate_naive, erode_fft,  # noqa: E402
                                 erode_naive)
from fftmorph.umbra import GridFunction  # noqa: E402

from paper_2305_03018_b200 import workloads as W  # noqa: E402


def out_digest(values, valid) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(values).astype(np.int32)).tobytes()
                          + np.ascontiguousarray(np.asarray(valid).astype(np.uint8)).tobytes()).hexdigest()


def grid(values, defined, lo, tonal_max):
    return GridFunction(values, defined, lo=lo, tonal_max=tonal_max)


def make_cases():
    rng = np.random.default_rng(20230503)
    arrays = {}
    meta = []
    n = 0
    for trial in range(120):
        nd = 1 if trial % 3 == 0 else 2
        if nd == 1:
            sh = (int(rng.integers(1, 90)),)
            ms = (int(rng.integers(1, 24)),)
        else:
            sh = tuple(int(x) for x in rng.integers(1, 40, 2))
            ms = tuple(int(x) for x in rng.integers(1, 12, 2))
        top = int(rng.choice([1, 7, 15, 31, 63, 255]))
        btop = int(rng.choice([0, 3, 7, 15]))
        gap_f = float(rng.choice([0.0, 0.0, 0.2]))
        gap_b = float(rng.choice([0.0, 0.3]))
        fv = rng.integers(0, top + 1, sh)
        fd = rng.random(sh) >= gap_f
        fd.flat[int(rng.integers(0, fd.size))] = True
        bv = rng.integers(0, btop + 1, ms)
        bd = rng.random(ms) >= gap_b
        bd.flat[int(rng.integers(0, bd.size))] = True
        f_lo = tuple(int(x) for x in rng.integers(-5, 6, nd))
        b_lo = tuple(int(-(m // 2) + rng.integers(-3, 4)) for m in ms)
        f = grid(fv, fd, f_lo, top)
        b = grid(bv, bd, b_lo, max(btop, 1))
        crop = bool(trial % 4 != 1)
        l = None if trial % 5 else top + int(rng.integers(0, 4))
        rec = {"nd": nd, "f_lo": f_lo, "b_lo": b_lo, "tonal_max": top, "b_tonal_max": max(btop, 1),
               "crop": crop, "l": l}
        key = f"c{n}"
        arrays[key + "_fv"] = fv
        arrays[key + "_fd"] = fd
        arrays[key + "_bv"] = bv
        arrays[key + "_bd"] = bd
        try:
            st = {}
            d, dv = dilate_fft(f, b, crop=crop, return_validity=True, stats=st)
            arrays[key + "_dil"] = d.values
            arrays[key + "_dilv"] = dv
            rec["dil_lo"] = d.lo
            rec["dil_tonal_max"] = d.tonal_max
            rec["dil_dev"] = st["max_abs_deviation"]
            dn, dnv = dilate_naive(f, b, crop=crop, return_validity=True)
            assert np.array_equal(dn.values, d.values) and np.array_equal(dnv, dv)
            rec["dil_error"] = None
        except Exception as e:  # the reference quirk (TypeError) is recorded
            rec["dil_error"] = type(e).__name__
        try:
            e_, ev = erode_fft(f, b, l=l, return_validity=True)
            arrays[key + "_ero"] = e_.values
            arrays[key + "_erov"] = ev
            rec["ero_lo"] = e_.lo
            rec["ero_tonal_max"] = e_.tonal_max
            rec["ero_error"] = None
        except Exception as e:
            rec["ero_error"] = type(e).__name__
        en, env = erode_naive(f, b, crop=crop, return_validity=True)
        arrays[key + "_eron"] = en.values
        arrays[key + "_eronv"] = env
        rec["eron_lo"] = en.lo
        meta.append(rec)
        n += 1
    np.savez_compressed(HERE / "cases.npz", **arrays)
    (HERE / "cases.json").write_text(json.dumps(meta, indent=0))
    print("cases:", n)


def make_small_configs():
    for name in ("c1", "c2"):
        w = W.CONFIGS[name]()
        f = GridFunction(w.images[0].astype(np.int64), tonal_max=w.tonal_max)
        b = GridFunction(w.se_values, w.se_defined, lo=w.se_lo, tonal_max=w.se_tonal_max)
        st = {}
        d, dv = dilate_fft(f, b, return_validity=True, stats=st)
        st2 = {}
        e, ev = erode_fft(f, b, return_validity=True, stats=st2)
        assert d == dilate_naive(f, b) and e == erode_naive(f, b)
        np.savez_compressed(HERE / f"{name}.npz", dil=d.values.astype(np.int16), dilv=dv,
                            ero=e.values.astype(np.int16), erov=ev,
                            dil_dev=st["max_abs_deviation"], ero_dev=st2["max_abs_deviation"],
                            padded=np.array(st["padded_shape"]))
        print(name, "dev", st["max_abs_deviation"], st2["max_abs_deviation"], st["padded_shape"])


def make_digests():
    out = {}
    jobs = [("c3", 0), ("c4", 0), ("c5", 0), ("c5", 1), ("c5", 63)]
    for name, i in jobs:
        if name == "c5":
            img = W.c5_image(i)
            w = W.c5(n_images=0) if False else None
            se, sd, lo, tm = W.c5_se(), np.ones((31, 31), bool), (-15, -15), 63
        else:
            w = W.CONFIGS[name]()
            img, se, sd, lo, tm = w.images[0], w.se_values, w.se_defined, w.se_lo, w.tonal_max
        f = GridFunction(img.astype(np.int64), tonal_max=tm)
        b = GridFunction(se, sd, lo=lo, tonal_max=max(int(se[sd].max()), 1))
        t = time.time()
        d, dv = dilate_naive(f, b, return_validity=True)
        e, ev = erode_naive(f, b, return_validity=True)
        key = f"{name}_img{i}"
        out[key] = {"dilate": out_digest(d.values, dv), "erode": out_digest(e.values, ev),
                    "input": W.digest(img), "dilate_valid_all": bool(dv.all()),
                    "erode_valid_all": bool(ev.all()),
                    "dilate_max": int(d.values.max()), "erode_min": int(e.values.min())}
        print(key, out[key], f"{time.time() - t:.1f}s", flush=True)
    (HERE / "digests.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    what = sys.argv[1:] or ["cases", "small", "digests"]
    if "cases" in what:
        make_cases()
    if "small" in what:
        make_small_configs()
    if "digests" in what:
        make_digests()
