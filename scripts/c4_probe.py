import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2305_03018_b200 import workloads as W
from paper_2305_03018_b200.engine import MorphPlan
w = W.c4()
plan = MorphPlan(shape=w.images.shape[1:], se_values=w.se_values, se_defined=w.se_defined, se_lo=w.se_lo,
                 mode="dilate", img_dtype=torch.uint8, img_min=0, img_max=15, batch=1)
x = torch.from_numpy(w.images).cuda()
for _ in range(3):
    plan.execute(x)
torch.cuda.synchronize()
print(plan.info)
