"""Time the c5 conv launches through the library's own event timing (A/B helper).

    FM_LIB=... python scripts/time_conv.py [--images 12] [--reps 3]
Prints conv/tonal/range ms per call; no correctness check (diagnostic variants).
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_03018_b200 import workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--images", type=int, default=12)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
imgs = np.stack([W.c5_image(i % 4) for i in range(a.images)])
plan = MorphPlan(shape=imgs.shape[1:], se_values=W.c5_se(), se_lo=(-15, -15), mode="dilate",
                 img_dtype=torch.uint8, img_min=0, img_max=63, fill=0, batch=a.images)
x = torch.from_numpy(imgs).cuda()
plan.execute(x)
torch.cuda.synchronize()
plan.set_timing(True)
plan.get_timing(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    plan.execute(x)
e1.record()
torch.cuda.synchronize()
t = plan.get_timing()
print(f"step_ms {e0.elapsed_time(e1) / a.reps:.3f} conv_ms {t['conv_ms'] / a.reps:.3f} tonal_ms {t['tonal_ms'] / a.reps:.3f}")
