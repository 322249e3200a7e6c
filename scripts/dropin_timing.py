"""Wall time of the drop-in API (numpy GridFunction in and out) on one c5 image."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_03018_b200 as fm  # noqa: E402
from paper_2305_03018_b200 import workloads as W  # noqa: E402

f = fm.GridFunction(W.c5_image(0).astype(np.int64), tonal_max=63)
b = fm.GridFunction(W.c5_se(), lo=(-15, -15), tonal_max=15)
for i in range(5):
    t0 = time.perf_counter()
    d = fm.dilate_fft(f, b)
    t1 = time.perf_counter()
    print(f"call {i}: {1e3 * (t1 - t0):.1f} ms  ({2048 * 2048 / (t1 - t0) / 1e6:.0f} Mpx/s)")
