"""Per-config device throughput (dilation and erosion) for the five BASELINE configs.

    python scripts/bench_configs.py [--images 8] [--reps 5]

Inputs resident in HBM, CUDA-event timed, warm plan (SE spectrum cached).
c5 uses --images images; the others one image (their BASELINE definition).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2305_03018_b200 import build, workloads as W  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402


def run(w, mode, reps):
    imgs = w.images
    dt = torch.int32 if imgs.dtype == np.int32 else torch.uint8
    plan = MorphPlan(shape=imgs.shape[1:], se_values=w.se_values, se_defined=w.se_defined, se_lo=w.se_lo,
                     mode=mode, img_dtype=dt, img_min=0, img_max=w.tonal_max,
                     fill=0 if mode == "dilate" else w.tonal_max, batch=imgs.shape[0])
    x = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
    out = torch.empty((imgs.shape[0], *plan.out_shape), dtype=torch.int32, device="cuda")
    valid = torch.empty_like(out, dtype=torch.uint8)
    for _ in range(2):
        plan.execute(x, out=out, valid=valid)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plan.reset_stats()
    e0.record()
    for _ in range(reps):
        plan.execute(x, out=out, valid=valid)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    dev = plan.read_stats()
    plan.set_timing(True)
    plan.execute(x, out=out, valid=valid)
    t = plan.get_timing(reset=True)
    plan.set_timing(False)
    px = int(np.prod(imgs.shape))
    return {"ms": ms, "mpix_s": px / ms / 1e3, "tile": plan.info["tile_x"], "T": plan.info["tonal_len"],
            "max_dev": dev, "range_ms": t["range_ms"], "conv_ms": t["conv_ms"], "tonal_ms": t["tonal_ms"],
            "conv_launches": t["conv_launches"], "tonal_launches": t["tonal_launches"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="c1,c2,c3,c4,c5")
    ap.add_argument("--modes", default="dilate,erode")
    args = ap.parse_args()
    build.build()
    res = {}
    for name in args.only.split(","):
        w = W.c5(n_images=args.images) if name == "c5" else W.CONFIGS[name]()
        for mode in args.modes.split(","):
            r = run(w, mode, args.reps)
            res[f"{name}_{mode}"] = r
            print(name, mode, json.dumps(r), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
