"""Stress one fuzz case: repeated runs with the device allocator pre-filled with
garbage (race / uninitialised-read hunting).  python scripts/stress_case.py SEED [reps]"""
import sys
import zlib
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import test_gpu_fuzz as T  # noqa: E402
from oracle import cnaive  # noqa: E402
from paper_2305_03018_b200.engine import MorphPlan  # noqa: E402

seed = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = T._case(zlib.crc32(f"fuzz/{seed}".encode()))
off = c["offset"]
img_min, img_max = off, off + c["levels"] - 1
fill = 0 if c["mode"] == "dilate" else img_max
tdt = {"uint8": torch.uint8, "uint16": torch.uint16, "int32": torch.int32}[c["dtype"]]
npdt = {"uint8": np.uint8, "uint16": np.uint16, "int32": np.int32}[c["dtype"]]
imgs = np.stack([np.roll(c["img"], i, axis=-1) for i in range(c["batch"])]) + off
defs = None if c["defined"] is None else np.stack([np.roll(c["defined"], i, axis=-1) for i in range(c["batch"])])
refs = [cnaive.naive(imgs[i], None if defs is None else defs[i], c["se"], c["se_def"], c["se_lo"],
                     erode=(c["mode"] == "erode"), crop=c["crop"], fill=fill) for i in range(c["batch"])]
fails = 0
for r in range(reps):
    junk = torch.full((int(3e9) // 4,), float(r + 0.5), dtype=torch.float32, device="cuda")
    del junk
    plan = MorphPlan(shape=c["shape"], se_values=c["se"], se_defined=c["se_def"], se_lo=c["se_lo"], mode=c["mode"],
                     crop=c["crop"], img_dtype=tdt, img_min=img_min, img_max=img_max, fill=fill,
                     batch=c["batch"], scratch_bytes=c["scratch"], tile=c["tile"])
    d = None if defs is None else torch.from_numpy(defs.astype(np.uint8)).cuda()
    out, valid = plan.execute(torch.from_numpy(imgs.astype(npdt)).cuda(), d)
    dev = plan.read_stats(raise_errors=False)
    bad = []
    for i in range(c["batch"]):
        o = out[i].cpu().numpy().astype(np.int64)
        diff = np.argwhere(o != refs[i][0].astype(np.int64))
        if len(diff):
            bad.append((i, len(diff), diff[:3].tolist()))
    if dev >= 0.25 or bad:
        fails += 1
        info = plan.info
        print("rep", r, "dev", dev, "bad", bad, "tile", info["tile_y"], info["tile_x"], "T", info["tonal_len"],
              "valid", info["valid_y"], info["valid_x"], "tiles", info["tiles_y"], info["tiles_x"])
    plan.close()
print(f"seed {seed}: {fails}/{reps} failed")
