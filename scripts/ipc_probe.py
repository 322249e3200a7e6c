"""c5 throughput vs images per launch (scratch budget) — how large is the per-launch tail?"""
import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_03018_b200 import workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402
n = 24
imgs = np.stack([W.c5_image(i % 8) for i in range(n)])
x = torch.from_numpy(imgs).cuda()
for gb in (2, 4, 8, 16):
    plan = MorphPlan(shape=(2048, 2048), se_values=W.c5_se(), se_lo=(-15, -15), img_dtype=torch.uint8, img_min=0,
                     img_max=63, batch=n, out_dtype=torch.uint8, scratch_bytes=gb << 30)
    out = torch.empty((n, 2048, 2048), dtype=torch.uint8, device="cuda")
    valid = torch.empty_like(out)
    for _ in range(2):
        plan.execute(x, out=out, valid=valid)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        plan.execute(x, out=out, valid=valid)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"scratch {gb} GiB: images/launch {plan.info['images_per_launch']}  {ms:.3f} ms  {n*4.194304/ms*1e3:.0f} Mpx/s", flush=True)
    del plan
