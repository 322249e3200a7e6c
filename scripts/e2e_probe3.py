"""Does a concurrent D2H/H2D copy stream slow the compute stream?  c5, 12 images."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_03018_b200 import workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

n = 12
imgs = np.stack([W.c5_image(i % 4) for i in range(n)])
plan = MorphPlan(shape=(2048, 2048), se_values=W.c5_se(), se_lo=(-15, -15), img_dtype=torch.uint8, img_min=0,
                 img_max=63, batch=n, out_dtype=torch.uint8)
x = torch.from_numpy(imgs).cuda()
dout = torch.empty((n, 2048, 2048), dtype=torch.uint8, device="cuda")
dvalid = torch.empty_like(dout)
big = torch.empty(400 << 20, dtype=torch.uint8, device="cuda")
pin = torch.empty(400 << 20, dtype=torch.uint8).pin_memory()
cs = torch.cuda.Stream()
ks = torch.cuda.Stream()


def run(copy_mode):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        c0.record()
        for _ in range(6):
            if copy_mode == "d2h":
                pin.copy_(big, non_blocking=True)
            elif copy_mode == "h2d":
                big.copy_(pin, non_blocking=True)
        c1.record()
    with torch.cuda.stream(ks):
        e0.record()
        plan.execute(x, out=dout, valid=dvalid, stream=ks)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), c0.elapsed_time(c1)


for mode in ("none", "d2h", "h2d", "none", "d2h"):
    print(mode, run(mode), flush=True)
