"""Run one BASELINE config once (dilation) — a target for ncu captures.

    python scripts/run_config_once.py c4 [--mode erode] [--reps 2]
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
ap.add_argument("name")
ap.add_argument("--mode", default="dilate")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--images", type=int, default=2)
a = ap.parse_args()
w = W.c5(n_images=a.images) if a.name == "c5" else W.CONFIGS[a.name]()
dt = torch.int32 if w.images.dtype == np.int32 else torch.uint8
plan = MorphPlan(shape=w.images.shape[1:], se_values=w.se_values, se_defined=w.se_defined, se_lo=w.se_lo,
                 mode=a.mode, img_dtype=dt, img_min=0, img_max=w.tonal_max,
                 fill=0 if a.mode == "dilate" else w.tonal_max, batch=w.images.shape[0])
x = torch.from_numpy(np.ascontiguousarray(w.images)).cuda()
for _ in range(a.reps):
    plan.execute(x)
torch.cuda.synchronize()
print("ok", plan.read_stats())
