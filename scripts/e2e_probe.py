"""Where does the host-buffer (e2e) path lose time against the device path?  c5 batch."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2305_03018_b200 import workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
imgs = np.stack([W.c5_image(i % 4) for i in range(n)])
se = W.c5_se()
plan = MorphPlan(shape=(2048, 2048), se_values=se, se_lo=(-15, -15), img_dtype=torch.uint8, img_min=0,
                 img_max=63, batch=n, out_dtype=torch.uint8)
x = torch.from_numpy(imgs).cuda()
pin_in = torch.from_numpy(imgs).pin_memory()
pin_out = torch.empty((n, 2048, 2048), dtype=torch.uint8).pin_memory()
pin_valid = torch.empty((n, 2048, 2048), dtype=torch.uint8).pin_memory()
dout = torch.empty((n, 2048, 2048), dtype=torch.uint8, device="cuda")
dvalid = torch.empty_like(dout)
s = torch.cuda.current_stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


print("device execute      ", timed(lambda: plan.execute(x, out=dout, valid=dvalid)))
print("execute_host        ", timed(lambda: plan.execute_host(pin_in, out=pin_out, valid=pin_valid)))
print("execute_host novalid", timed(lambda: plan.execute_host(pin_in, out=pin_out, want_valid=False)))
print("H2D only            ", timed(lambda: x.copy_(pin_in, non_blocking=True)))
print("D2H only (out+valid)", timed(lambda: (pin_out.copy_(dout, non_blocking=True), pin_valid.copy_(dvalid, non_blocking=True))))
