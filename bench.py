"""Benchmark of the hot path: exact FFT dilation of the BASELINE c5 batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU)

Workload (BASELINE.json configs[4], the metric's 1/2/4/8-GPU config): 64
images of 2048x2048, 6-bit smooth noise (SURVEY.md §8(d) recipe, seeded), a
31x31 non-flat SE with offsets in [0,15]; exact dilation; the 64 images are
sharded by image across ranks (no collective on the data path).  A step is
one pass of the hot path over the rank's images, inputs resident in HBM.

--impl reference times the reference's algorithm on the host CPU
(oracle/port.py, a restatement of fftmorph.dilate_fft: tonal one-hot volumes,
scipy real FFTs with all host threads, projection) on a bounded 512x512 crop
sample of the same workload — the reference package itself is pure Python
and cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "exact dilation output Mpixel/s"
UNIT = "Mpixel/s"
N_IMAGES = 64
EDGE = 2048


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _ncu_traffic(images_per_launch):
    """DRAM bytes per conv launch from the newest committed ncu capture of this workload
    (profiles/r*_c5_tile_conv_tonal.json, written by scripts/ncu_summary.py)."""
    files = sorted((ROOT / "profiles").glob("r*_c5_tile_conv_tonal.json"), key=lambda f: f.name)
    for f in reversed(files):
        try:
            data = json.loads(f.read_text())
        except Exception:
            continue
        for k in data.get("kernels", []):
            name = k["kernel"]
            if (name.startswith("void tile128_kernel<") and not name.endswith("1>(TileArgs)")
                    and "dram_bytes_per_launch" in k):
                ipl = data.get("images_per_launch", 4)
                pipe = {"fma_pipe_active": k.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                        "issue_active": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                        "shared_wavefronts": k.get(
                            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")}
                return k["dram_bytes_per_launch"] * images_per_launch / ipl, f.name, pipe
    return None, None, None


def method_floor(mpx_s, hbm_gbs):
    """SURVEY §8(d) B_alg/px = [|F| (s_in + 4) + 8 V] / |F|, V = S_lin (l_R + 1), for the c5
    workload (l_R = 63 + 15, full-mode S_lin = (2048 + 30)^2, uint8 in, int32 out), and the
    path's fraction of HBM at that algorithmic traffic."""
    f = EDGE * EDGE
    v = (EDGE + 30) ** 2 * (63 + 15 + 1)
    b_alg = (f * (1 + 4) + 8.0 * v) / f
    achieved = b_alg * mpx_s * 1e6 / 1e9
    return {"bytes_per_px": b_alg, "achieved_gbs": achieved, "peak_gbs": hbm_gbs, "frac": achieved / hbm_gbs}


def _gen(i):
    from paper_2305_03018_b200 import workloads as W
    return W.c5_image(i)


def make_images(idx):
    idx = list(idx)
    if not idx:
        return np.zeros((0, EDGE, EDGE), np.uint8)
    workers = max(1, min(len(idx), len(os.sched_getaffinity(0)), 32))
    with ProcessPoolExecutor(workers) as ex:
        return np.stack(list(ex.map(_gen, idx)))


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.proc = None
        self.path = Path(f"/tmp/fm_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def wait_first(self, timeout=10.0):
        """Block until nvidia-smi has written its first sample (its start-up takes longer
        than a short timed region)."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout:
            try:
                if self.path.stat().st_size > 0:
                    return
            except FileNotFoundError:
                pass
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
            except ValueError:
                continue
        try:
            self.path.unlink()
        except Exception:
            pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3]) if v.lower() == "active"})
        loaded = [r for r in rows if r[2] > 200.0] or rows
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "power_w_max": max(r[2] for r in rows), "reasons": reasons}


def cpu_reference(seconds_target=(10.0, 30.0), sample_edge=512, steps=None, warmup=0):
    """Time oracle/port.dilate_fft (the reference's algorithm) on crops of c5 image 0."""
    from oracle import port
    from paper_2305_03018_b200 import workloads as W
    cores = len(os.sched_getaffinity(0))
    img = W.c5_image(0)
    se = W.c5_se()
    crops = [img[y:y + sample_edge, x:x + sample_edge] for y in range(0, EDGE, sample_edge)
             for x in range(0, EDGE, sample_edge)]
    for i in range(warmup):
        port.dilate_fft(crops[i % len(crops)], None, (0, 0), se, None, (-15, -15), workers=cores)
    times = []
    n = 0
    t_all = time.perf_counter()
    while True:
        c = crops[n % len(crops)]
        t0 = time.perf_counter()
        port.dilate_fft(c, None, (0, 0), se, None, (-15, -15), workers=cores)
        times.append(time.perf_counter() - t0)
        n += 1
        if steps is not None:
            if n >= steps:
                break
        elif time.perf_counter() - t_all >= seconds_target[0] or n >= len(crops):
            break
    px = sample_edge * sample_edge
    return {"value": px * n / sum(times) / 1e6, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n} x {sample_edge}x{sample_edge} crops of c5 image 0, oracle/port.dilate_fft "
                      f"(reference algorithm: int64 umbra, scipy rfftn/irfftn workers={cores}, project)",
            "seconds": sum(times), "steps_s": times}


def run_reference(args, rank, world):
    if rank != 0:
        return
    res = cpu_reference(steps=args.steps, warmup=args.warmup)
    ms = 1000.0 * sum(res["steps_s"]) / len(res["steps_s"])
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8(d) c5 recipe)",
        "config": {"workload": "c5 sample: 512x512 crop of a 2048x2048 6-bit image, 31x31 SE [0,15], dilation"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2305_03018_b200 import _lib
    from paper_2305_03018_b200 import build as B
    from paper_2305_03018_b200 import workloads as W
    from paper_2305_03018_b200.engine import MorphPlan
    from paper_2305_03018_b200.sharding import shard_range

    B.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    i0, i1 = shard_range(args.images, rank, world)
    nloc = i1 - i0
    imgs = make_images(range(i0, i1))
    se = W.c5_se()
    # dilation values of c5 lie in [0, 63 + 15]: the plan checks they fit the output type
    out_dt = {"u8": torch.uint8, "i16": torch.int16, "i32": torch.int32}[args.out_dtype]
    plan = MorphPlan(shape=(EDGE, EDGE), se_values=se, se_lo=(-15, -15), mode="dilate", crop=True,
                     img_dtype=torch.uint8, img_min=0, img_max=63, fill=0, batch=max(nloc, 1),
                     device=dev, scratch_bytes=args.scratch_gib << 30, out_dtype=out_dt)
    x = torch.from_numpy(imgs).to(dev)
    out = torch.empty((nloc, EDGE, EDGE), dtype=out_dt, device=dev)
    valid = torch.empty((nloc, EDGE, EDGE), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.execute(x, out=out, valid=valid, stream=stream)

    # the clock sampler runs from before the warm-up (all of it under load) to the end
    # of the timed region
    clocks = Clocks(local_rank)
    clocks.wait_first()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.reset_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    plan.get_timing(reset=True)
    plan.set_timing(True)
    l0 = _lib.kernel_launches()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        step()
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = _lib.kernel_launches() - l0
    plan.set_timing(False)
    clk = clocks.stop()
    ms = start.elapsed_time(stop)
    tim = plan.get_timing(reset=True)
    dev_max = plan.read_stats()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    ms_per_step = ms_max / args.steps
    mpx = args.images * EDGE * EDGE / 1e6
    value = mpx / (ms_per_step / 1000.0)

    # e2e: same metric through the public API with HOST buffers (pinned), copies inside
    pin_in = torch.from_numpy(imgs).pin_memory()
    pin_out = torch.empty((nloc, EDGE, EDGE), dtype=out_dt).pin_memory()
    pin_valid = torch.empty((nloc, EDGE, EDGE), dtype=torch.uint8).pin_memory()
    plan.execute_host(pin_in, out=pin_out, valid=pin_valid, stream=stream)   # warm (staging alloc)
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        plan.execute_host(pin_in, out=pin_out, valid=pin_valid, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    wall_ms = (time.perf_counter() - t0) * 1000.0 / e2e_steps
    e2e_t = torch.tensor([max(e2e_ms, wall_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_val = mpx / (float(e2e_t.item()) / 1000.0)

    if rank != 0:
        return
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs")
    peak_note = "measured (MEASURED_PEAKS.json)" if hbm else "fallback (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    conv_s = tim["conv_ms"] / 1000.0 / max(tim["conv_launches"], 1)
    conv_bytes = tim["conv_bytes"] / max(tim["conv_launches"], 1)
    achieved = conv_bytes / conv_s / 1e9 if conv_s > 0 else 0.0
    tonal_s = tim["tonal_ms"] / 1000.0 / max(tim["tonal_launches"], 1)
    tonal_bytes = tim["tonal_bytes"] / max(tim["tonal_launches"], 1)
    sm_mhz = (clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    conv_tflops = tim["conv_flops"] / max(tim["conv_launches"], 1) / conv_s / 1e12 if conv_s > 0 else 0.0
    info = plan.info
    traffic, traffic_src, pipe = _ncu_traffic(info["images_per_launch"])
    fpp = 2.0 * 5.0 * 128 * 128 * math.log2(128 * 128) + 6.0 * 128 * 128
    tiles = info["tiles_y"] * info["tiles_x"]
    mean_planes = tim["conv_flops"] / fpp / (tiles * args.images * args.steps) if tim["conv_flops"] else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SURVEY §8(d) c5 recipe, seeded PCG64)",
        "config": {"workload": f"c5: {args.images} x {EDGE}x{EDGE} 6-bit smooth-noise images, 31x31 non-flat SE "
                               "[0,15], exact dilation, sharded by image",
                   "images": args.images, "images_per_gpu": nloc, "tonal_len": info["tonal_len"],
                   "planes_max": info["planes"], "mean_planes_per_tile": mean_planes,
                   "tile": [info["tile_y"], info["tile_x"]], "tiles_per_image": tiles,
                   "window": [info["valid_y"], info["valid_x"]],
                   "images_per_launch": info["images_per_launch"],
                   "l2": "no flush: inputs 256 MiB and the spectral volume (~0.7 GB/image at "
                         f"{(mean_planes or 0):.1f} planes/tile) exceed the 126 MB L2"},
        "roofline": {"bound": "hbm", "kernel": "tile128_kernel (encode + three-pass 2-D FFT conv, fm_tile128.cuh)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_note,
                     "bytes_per_launch": conv_bytes, "ms_per_launch": conv_s * 1000.0,
                     "fp32_tflops_nominal": conv_tflops, "fp32_peak_tflops_at_sm_mhz": fp32_peak,
                     "fp32_frac": conv_tflops / fp32_peak if fp32_peak else None,
                     # what actually bounds the conv kernel (ncu, same capture as traffic, % of peak)
                     "limiter": "FMA pipe (packed f32x2 FFT butterflies) + shared-memory exchanges; not HBM",
                     "ncu_pct": pipe,
                     "tonal_kernel": {"achieved": tonal_bytes / tonal_s / 1e9 if tonal_s > 0 else 0.0,
                                      "unit": "GB/s", "frac": (tonal_bytes / tonal_s / 1e9) / hbm if tonal_s > 0 else 0.0,
                                      "ms_per_launch": tonal_s * 1000.0},
                     # the range kernels run one launch chunk ahead on a low-priority stream
                     # (overlapping the conv tail / tonal kernels): their event span is not a
                     # share of the step
                     "share_of_step": {"conv": tim["conv_ms"] / max(ms, 1e-9), "tonal": tim["tonal_ms"] / max(ms, 1e-9)},
                     # the whole path against the method's HBM floor (spectral volume of
                     # minimal extent S_lin x (l_R + 1) written once and read once, plus the image I/O)
                     "method_floor": method_floor(value, hbm)},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(imgs.nbytes),
                "d2h_bytes_per_step": int(pin_out.numel() * pin_out.element_size() + pin_valid.numel())},
        "gpu_launches": int(launches),
        "max_abs_deviation": dev_max,
        "clocks": clk,
    }
    if args.cpu_baseline and world == 1:
        try:
            cb = cpu_reference()
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # keep the GPU line even if the host baseline fails (e.g. RAM)
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                                    "kind": "port", "sample": f"failed: {type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--images", type=int, default=N_IMAGES)
    ap.add_argument("--scratch-gib", type=int, default=16)
    ap.add_argument("--out-dtype", choices=["u8", "i16", "i32"], default="u8",
                    help="output value type (the c5 dilation range 0..78 fits u8)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
