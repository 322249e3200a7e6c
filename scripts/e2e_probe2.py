"""e2e overhead vs batch size (c5 images): device execute vs execute_host."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_03018_b200 import workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

base = np.stack([W.c5_image(i) for i in range(4)])
se = W.c5_se()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in (3, 6, 12, 24):
    imgs = np.stack([base[i % 4] for i in range(n)])
    plan = MorphPlan(shape=(2048, 2048), se_values=se, se_lo=(-15, -15), img_dtype=torch.uint8, img_min=0,
                     img_max=63, batch=n, out_dtype=torch.uint8)
    x = torch.from_numpy(imgs).cuda()
    pin_in = torch.from_numpy(imgs).pin_memory()
    pin_out = torch.empty((n, 2048, 2048), dtype=torch.uint8).pin_memory()
    pin_valid = torch.empty((n, 2048, 2048), dtype=torch.uint8).pin_memory()
    dout = torch.empty((n, 2048, 2048), dtype=torch.uint8, device="cuda")
    dvalid = torch.empty_like(dout)
    d = timed(lambda: plan.execute(x, out=dout, valid=dvalid))
    h = timed(lambda: plan.execute_host(pin_in, out=pin_out, valid=pin_valid))
    hn = timed(lambda: plan.execute_host(pin_in, out=pin_out, want_valid=False))
    dn = timed(lambda: plan.execute(x, out=dout, want_valid=False))
    print(f"n={n:3d} device {d:8.3f}  host {h:8.3f} (+{h-d:6.3f})  device-novalid {dn:8.3f} host-novalid {hn:8.3f} (+{hn-dn:6.3f})", flush=True)
    del plan
