"""The reference's acceptance criteria 3 and 4 (test_acceptance.py:110-137) as reported
characteristics of the B200 path (CPU timing trends, not parity gates).

    python scripts/acceptance_trends.py

Criterion 3: 256x256 4-bit image, flat square SEs 16..96 wide: time(96) / time(16) of the FFT
method (reference: < 1.5) and of the naive method (reference: > 5).  Criterion 4: 128x128
image, flat 13x13 SE: 8-bit / 4-bit time ratio of the FFT method (reference: in [4, 40]).
Same calls as the reference test (drop-in API, numpy grids in and out, best of n); the
device-resident plan time is printed beside it."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_03018_b200 as fm  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402


def best_of(n, fn):
    best = float("inf")
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def device_ms(img, se, vmax, reps=20):
    plan = MorphPlan(shape=img.shape, se_values=se, se_lo=tuple(-(s // 2) for s in se.shape), mode="dilate",
                     img_dtype=torch.uint8, img_min=0, img_max=vmax, fill=0, batch=1)
    x = torch.from_numpy(img.astype(np.uint8)[None]).cuda()
    for _ in range(3):
        plan.execute(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.execute(x)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    rng = np.random.default_rng(2000)
    f_np = rng.integers(0, 16, (256, 256))
    f = fm.GridFunction(f_np, tonal_max=15)
    t, dev = {}, {}
    for width in (16, 32, 48, 64, 80, 96):
        se = np.zeros((width, width), np.int64)
        b = fm.GridFunction(se, lo=(-(width // 2), -(width // 2)), tonal_max=1)
        for method, fn in (("fft", fm.dilate_fft), ("naive", fm.dilate_naive)):
            fn(f, b)   # plan / first-call costs
            t[method, width] = best_of(3, lambda: fn(f, b))
        dev[width] = device_ms(f_np, se, 15)
    print("criterion 3 (256x256 4-bit, flat SE width 16..96), drop-in call ms:")
    for width in (16, 32, 48, 64, 80, 96):
        print(f"  width {width:3d}: fft {1e3 * t['fft', width]:.3f}  naive {1e3 * t['naive', width]:.3f}  "
              f"device-resident fft {dev[width]:.3f}")
    print(f"  fft ratio 96/16: {t['fft', 96] / t['fft', 16]:.2f} (reference CPU: < 1.5; device-resident "
          f"{dev[96] / dev[16]:.2f}), naive ratio {t['naive', 96] / t['naive', 16]:.1f} (reference CPU: > 5)")
    rng = np.random.default_rng(3000)
    se = np.zeros((13, 13), np.int64)
    b = fm.GridFunction(se, lo=(-6, -6), tonal_max=1)
    t4, d4 = {}, {}
    for bits in (4, 8):
        vmax = (1 << bits) - 1
        f_np = rng.integers(0, vmax + 1, (128, 128))
        f = fm.GridFunction(f_np, tonal_max=vmax)
        fm.dilate_fft(f, b)
        t4[bits] = best_of(5, lambda: fm.dilate_fft(f, b))
        d4[bits] = device_ms(f_np, se, vmax)
    print(f"criterion 4 (128x128, flat 13x13 SE): 4-bit {1e3 * t4[4]:.3f} ms, 8-bit {1e3 * t4[8]:.3f} ms, ratio "
          f"{t4[8] / t4[4]:.2f} (reference CPU: in [4, 40]); device-resident {d4[4]:.3f} / {d4[8]:.3f} ms, "
          f"ratio {d4[8] / d4[4]:.2f}")


if __name__ == "__main__":
    main()
