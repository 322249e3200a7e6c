"""cProfile of the drop-in call on a small config: python scripts/dropin_profile.py [c1|c2] [calls]"""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_03018_b200 as fm  # noqa: E402
from paper_2305_03018_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 300
w = W.CONFIGS[name]()
f = fm.GridFunction(w.images[0].astype("int64"), tonal_max=w.tonal_max)
b = fm.GridFunction(w.se_values, w.se_defined, lo=w.se_lo, tonal_max=w.se_tonal_max)
for _ in range(5):
    fm.dilate_fft(f, b)
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    fm.dilate_fft(f, b)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(28)
