"""the reference algorithm timed on this box's host cores.

    python scripts/cpu_baseline_table.py [--skip-naive-c4] > table.md

oracle/port (the line-by-line restatement of fftmorph.morphology.dilate_fft / erode_fft /
dilate_naive: int64 umbra volumes, scipy rfftn / irfftn in f64, rint, projection) on the seeded
inputs of SURVEY 8(d): c1..c4 with n = every host core and n = 1 FFT workers (best of 3 for
c1 / c2, one run for c3 / c4), the first images of c5 with the x16 extrapolation to the batch,
and the exact naive path (dilate_naive).  perf_counter brackets the call only; inputs pre-built.
Peak RSS is the process maximum so far (the calls run serially, largest last)."""
import argparse
import json
import os
import platform
import resource
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import port  # noqa: E402
from paper_2305_03018_b200 import workloads as W  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def timed(fn, reps):
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-naive-c4", action="store_true", help="dilate_naive at c4 takes ~2 min")
    ap.add_argument("--c5-images", type=int, default=2)
    args = ap.parse_args()
    cores = len(os.sched_getaffinity(0))
    rows = []

    def add(cfg, op, workers, secs, px, note=""):
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
        rows.append({"cfg": cfg, "op": op, "workers": workers, "s": secs, "mpix_s": px / secs / 1e6,
                     "rss_gib": rss, "note": note})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)

    for name in ("c1", "c2", "c4", "c3"):
        w = W.CONFIGS[name]()
        img, se, sd, lo, l = w.images[0], w.se_values, w.se_defined, w.se_lo, w.tonal_max
        z = (0,) * img.ndim
        reps = 3 if name in ("c1", "c2") else 1
        for n in (cores, 1):
            add(name, "dilate_fft", n, timed(lambda: port.dilate_fft(img, None, z, se, sd, lo, workers=n), reps), img.size,
                f"best of {reps}" if reps > 1 else "1 run")
            add(name, "erode_fft", n, timed(lambda: port.erode_fft(img, None, z, se, sd, lo, l=l, workers=n), reps), img.size,
                f"best of {reps}" if reps > 1 else "1 run")
        if name != "c4" or not args.skip_naive_c4:
            add(name, "dilate_naive", "-", timed(lambda: port.dilate_naive(img, None, z, se, sd, lo), 1), img.size, "exact path")
    se5 = W.c5_se()
    for i in range(args.c5_images):
        img = W.c5_image(i)
        add("c5", f"dilate_fft img{i}", cores,
            timed(lambda: port.dilate_fft(img, None, (0, 0), se5, None, (-15, -15), workers=cores), 1), img.size,
            "x64 images = batch")
    img = W.c5_image(0)
    add("c5", "erode_fft img0", cores,
        timed(lambda: port.erode_fft(img, None, (0, 0), se5, None, (-15, -15), l=63, workers=cores), 1), img.size)
    add("c5", "dilate_naive img0", "-", timed(lambda: port.dilate_naive(img, None, (0, 0), se5, None, (-15, -15)), 1),
        img.size, "exact path")

    c5 = [r for r in rows if r["cfg"] == "c5" and r["op"].startswith("dilate_fft")]
    per = sum(r["s"] for r in c5) / len(c5)
    print(f"# Reference algorithm on the host cores ({cores} x {cpu_model()}, numpy {np.__version__})\n")
    print("| cfg | op | FFT workers | wall s | output Mpixel/s | peak RSS so far (GiB) | note |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['cfg']} | {r['op']} | {r['workers']} | {r['s']:.3f} | {r['mpix_s']:.4g} | {r['rss_gib']:.1f} | {r['note']} |")
    print(f"\nc5 batch of 64 images, extrapolated from {len(c5)} image(s): {per:.1f} s per image, "
          f"{64 * per / 60:.1f} min for the batch ({4.194304 / per:.3f} Mpixel/s).")


if __name__ == "__main__":
    main()
