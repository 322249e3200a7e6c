import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2305_03018_b200.engine import MorphPlan
rng = np.random.default_rng(1)
img = rng.integers(0, 64, (200, 180))
se = rng.integers(0, 16, (31, 31))
plan = MorphPlan(shape=img.shape, se_values=se, se_lo=(-15, -15), mode="dilate", img_dtype=torch.uint8,
                 img_min=0, img_max=63, fill=0, batch=1)
out, valid = plan.execute(torch.from_numpy(img.astype(np.uint8)[None]).cuda())
print("dev", plan.read_stats())
