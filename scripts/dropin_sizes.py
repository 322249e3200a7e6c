"""Drop-in call time (numpy grids in and out) over image sizes: python scripts/dropin_sizes.py"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_03018_b200 as fm  # noqa: E402

rng = np.random.default_rng(1)
b = fm.GridFunction(rng.integers(0, 4, (9, 9)), lo=(-4, -4), tonal_max=3)
for n in (32, 64, 128, 192, 256, 384, 512, 1024):
    f = fm.GridFunction(rng.integers(0, 32, (n, n)), tonal_max=31)
    ts = []
    for i in range(25):
        t0 = time.perf_counter()
        fm.dilate_fft(f, b)
        ts.append(time.perf_counter() - t0)
    print(f"{n:5d}^2  median {1e6 * sorted(ts[3:])[len(ts[3:]) // 2]:8.0f} us")
