"""Digests of the exact c5 outputs for ALL 64 benchmarked images (dilation and erosion).

    python tests/golden/make_c5_digests.py            # -> tests/golden/c5_all_digests.json

The checker is the C restatement of dilate_naive / erode_naive (oracle/naive.c,
morphology.py:65-113), which is itself pinned to the REFERENCE: for images 0, 1
and 63 its digests must equal the ones `make_golden.py` recorded by running the
reference's own dilate_naive / erode_naive (digests.json) — this script asserts
that before writing anything.  The digest recipe is the same as make_golden.py:
sha256(int32 values || uint8 validity) over the 2048x2048 output.

Inputs follow SURVEY §8(d) (paper_2305_03018_b200.workloads.c5_image / c5_se).
Used by tests/test_gpu_bench_parity.py and by bench.py's post-timing parity check.
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

from oracle import cnaive  # noqa: E402
from paper_2305_03018_b200 import workloads as W  # noqa: E402


def out_digest(values, valid) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(values).astype(np.int32)).tobytes()
                          + np.ascontiguousarray(np.asarray(valid).astype(np.uint8)).tobytes()).hexdigest()


def main(n_images: int = 64) -> None:
    pinned = json.loads((HERE / "digests.json").read_text())
    se = W.c5_se()
    lo = (-15, -15)
    out = {"recipe": "sha256(int32 values || uint8 validity), 2048x2048, crop=True; "
                     "dilate_naive (fill 0) / erode_naive (neutral = tonal_max 63)",
           "checker": "oracle/naive.c, pinned to the reference's digests for images 0, 1, 63",
           "images": {}}
    for i in range(n_images):
        t = time.time()
        img = W.c5_image(i)
        d, dv = cnaive.naive(img, None, se, None, lo, erode=False, crop=True, fill=0)
        e, ev = cnaive.naive(img, None, se, None, lo, erode=True, crop=True, fill=63)
        rec = {"input": W.digest(img), "dilate": out_digest(d, dv), "erode": out_digest(e, ev),
               "dilate_max": int(d.max()), "erode_min": int(e.min()),
               "valid_all": bool(dv.all() and ev.all())}
        ref = pinned.get(f"c5_img{i}")
        if ref is not None:   # pin the checker to the reference's own outputs
            assert ref["input"] == rec["input"], (i, "input digest")
            assert ref["dilate"] == rec["dilate"] and ref["erode"] == rec["erode"], (i, "oracle != reference")
            rec["pinned_to_reference"] = True
        out["images"][str(i)] = rec
        print(i, rec["dilate"][:16], rec["erode"][:16], f"{time.time() - t:.1f}s", flush=True)
    (HERE / "c5_all_digests.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
