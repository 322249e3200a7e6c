import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import random_grid
import paper_2305_03018_b200 as m
from paper_2305_03018_b200.engine import MorphPlan
import torch
rng = np.random.default_rng(2000)
runs = 0
for bits in (1, 2, 4, 6, 8):
    top = (1 << bits) - 1
    for edge in (7, 33, 64, 130):
        for fe in (1, 3, 5, 9, 17):
            if fe > edge: continue
            f = random_grid(rng, (edge, edge), top, gap_p=0.1 if runs % 3 == 0 else 0.0)
            sev = rng.integers(0, top + 1, (fe, fe)) if runs % 2 else np.zeros((fe, fe), np.int64)
            b = m.GridFunction(sev, lo=(-(fe // 2), -(fe // 2)), tonal_max=max(top, 1))
            print("case", bits, edge, fe, runs, "gaps" if runs % 3 == 0 else "", flush=True)
            d, dv = m.dilate_fft(f, b, return_validity=True)
            e = m.erode_fft(f, b)
            runs += 1
print("ok")
