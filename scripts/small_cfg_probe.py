import sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2305_03018_b200 import workloads as W
from paper_2305_03018_b200.engine import MorphPlan
for name in ("c2", "c1"):
    w = W.CONFIGS[name]()
    dt = torch.int32 if w.images.dtype == np.int32 else torch.uint8
    for tile in ((0, 64, 128, 32) if name == "c2" else (0, 64, 128, 256)):
        try:
            plan = MorphPlan(shape=w.images.shape[1:], se_values=w.se_values, se_defined=w.se_defined, se_lo=w.se_lo,
                             mode="dilate", img_dtype=dt, img_min=0, img_max=w.tonal_max, fill=0,
                             batch=w.images.shape[0], tile=tile)
        except Exception as e:
            print(name, tile, "n/a", e); continue
        x = torch.from_numpy(np.ascontiguousarray(w.images)).cuda()
        for _ in range(5): plan.execute(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        for _ in range(50): plan.execute(x)
        e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(name, "tile", tile, "->", plan.info["tile_x"], f"gpu {e0.elapsed_time(e1)/50*1000:.1f} us  wall {(t1-t0)/50*1e6:.1f} us")
