"""Stress a synthetic case shaped like fuzz seed 124 with a chosen level count
(T > 254 -> uint16 tile kernel, else uint8): python scripts/stress_custom.py LEVELS REPS [gaps]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import cnaive  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

levels = int(sys.argv[1]); reps = int(sys.argv[2]); gaps = len(sys.argv) < 4 or sys.argv[3] != "nogaps"
rng = np.random.default_rng(124)
shape = (475, 519)
img = rng.integers(0, levels, shape)
defined = (rng.random(shape) > 0.46) if gaps else None
se = rng.integers(0, 2, (58, 33))
fails = 0
for r in range(reps):
    junk = torch.full((int(2e9) // 4,), float(r + 0.5), dtype=torch.float32, device="cuda")
    del junk
    plan = MorphPlan(shape=shape, se_values=se, se_lo=(-3, -3), mode="dilate", img_dtype=torch.int32,
                     img_min=0, img_max=levels - 1, fill=0, batch=3)
    imgs = np.stack([np.roll(img, i, axis=-1) for i in range(3)])
    defs = None if defined is None else np.stack([np.roll(defined, i, axis=-1) for i in range(3)])
    d = None if defs is None else torch.from_numpy(defs.astype(np.uint8)).cuda()
    out, valid = plan.execute(torch.from_numpy(imgs.astype(np.int32)).cuda(), d)
    dev = plan.read_stats(raise_errors=False)
    ok = dev < 0.25
    if ok:
        ref, rv = cnaive.naive(imgs[0], None if defs is None else defs[0], se, None, (-3, -3))
        ok = np.array_equal(out[0].cpu().numpy().astype(np.int64), ref.astype(np.int64))
    if not ok:
        fails += 1
        print("rep", r, "dev", dev, "T", plan.info["tonal_len"], "tile", plan.info["tile_x"])
print(f"levels {levels} gaps {gaps}: {fails}/{reps} failed (T={plan.info['tonal_len']})")
