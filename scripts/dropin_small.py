"""Wall time of the drop-in API (numpy GridFunction in and out) on the small configs c1 / c2."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_03018_b200 as fm  # noqa: E402
from paper_2305_03018_b200 import workloads as W  # noqa: E402

for name in ("c1", "c2"):
    w = W.CONFIGS[name]()
    f = fm.GridFunction(w.images[0].astype("int64"), tonal_max=w.tonal_max)
    b = fm.GridFunction(w.se_values, w.se_defined, lo=w.se_lo, tonal_max=w.se_tonal_max)
    ts = []
    for i in range(30):
        t0 = time.perf_counter()
        fm.dilate_fft(f, b)
        ts.append(time.perf_counter() - t0)
    print(name, "first", f"{1e3 * ts[0]:.2f} ms", "median of the rest", f"{1e6 * sorted(ts[1:])[len(ts) // 2]:.0f} us")
