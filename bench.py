"""Benchmark of the hot path: exact FFT dilation of the BASELINE c5 batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU)

Workload (BASELINE.json configs[4], the metric's 1/2/4/8-GPU config): 64
images of 2048x2048, 6-bit smooth noise (SURVEY.md §8(d) recipe, seeded), a
31x31 non-flat SE with offsets in [0,15]; exact dilation; the 64 images are
sharded by image across ranks (no collective on the data path).  A step is
one pass of the hot path over the rank's images, inputs resident in HBM.
After the timed region every output image (device-resident run, host-buffer
run, and the erosion run) is checked bit-exact against the committed
reference digests (tests/golden/c5_all_digests.json) -> "parity".

--impl reference times the reference's algorithm on the host CPU
(oracle/port.py, a restatement of fftmorph.dilate_fft: tonal one-hot volumes,
scipy real FFTs in f64 with all host threads, projection) on FULL 2048x2048
c5 images, one per step -- the reference package itself is pure Python and
cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
import hashlib
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
WORKLOAD = ("c5: 64 x 2048x2048 6-bit smooth-noise images, 31x31 non-flat SE [0,15], exact dilation, "
            "sharded by image")
WORKLOADS = {
    "c5": WORKLOAD,
    "c3": "c3: 1024x1024 8-bit blob image, 21x21 disk SE [0,7], exact dilation, row strips with SE halos",
    "c4": "c4: 2048x2048 4-bit image, 101x101 random flat mask SE, exact dilation, row strips with SE halos",
}
GOLDEN = ROOT / "tests" / "golden" / "c5_all_digests.json"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def _ncu_traffic(images_per_launch, images):
    """From the newest committed ncu capture of this workload (profiles/r*_c5_tile_conv_tonal.json,
    written by scripts/ncu_summary.py): DRAM bytes per conv launch scaled to this launch size, the
    conv kernel's pipe utilisation, and DRAM bytes per step (every captured kernel's bytes per
    image, summed, times the step's images)."""
    files = sorted((ROOT / "profiles").glob("r*_c5_tile_conv_tonal.json"), key=lambda f: f.name)
    for f in reversed(files):
        try:
            data = json.loads(f.read_text())
        except Exception:
            continue
        ipl = data.get("images_per_launch", 4)
        conv = None
        for k in data.get("kernels", []):
            name = k["kernel"]
            if (name.startswith("void tile128_kernel<") and not name.endswith("1>(TileArgs)")
                    and "dram_bytes_per_launch" in k):
                conv = k
        if conv is None:
            continue
        pipe = {"fma_pipe_active": conv.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                "issue_active": conv.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "shared_wavefronts": conv.get(
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")}
        step = data.get("dram_bytes_per_image")
        return (conv["dram_bytes_per_launch"] * images_per_launch / ipl, f.name, pipe,
                None if step is None else step * images)
    return None, None, None, None


def _fp32_peak(sm_mhz):
    """FP32 FMA peak at the measured SM clock: the microbenchmarked per-clock rate
    (profiles/*_fp32_peak.json, scripts/micro/ffma2_rate.cu) when committed, else the
    derived 148 SM x 128 lanes x 2 flop per clock."""
    files = sorted((ROOT / "profiles").glob("r*_fp32_peak.json"), key=lambda f: f.name)
    for f in reversed(files):
        try:
            d = json.loads(f.read_text())
            return d["flops_per_clock"] * sm_mhz * 1e6 / 1e12, f"measured per clock ({f.name}) x clock"
        except Exception:
            continue
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12, "derived: 148 SM x 128 FP32 lanes x 2 flop x SM clock"


def method_floor(mpx_s, hbm_gbs, out_bytes=4):
    """SURVEY §8(d) B_alg/px = [|F| (s_in + s_out) + 8 V] / |F|, V = S_lin (l_R + 1), for the c5
    workload (l_R = 63 + 15, full-mode S_lin = (2048 + 30)^2, uint8 in), and the path's
    EFFECTIVE fraction of HBM at that algorithmic traffic (the per-tile tonal length moves less
    than the floor's volume, so this is not a measured bandwidth)."""
    f = EDGE * EDGE
    v = (EDGE + 30) ** 2 * (63 + 15 + 1)
    b_alg = (f * (1 + out_bytes) + 8.0 * v) / f
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


def cpu_reference(steps=1, warmup=0, op="dilate", config="c5", budget_s=None):
    """Time oracle/port.dilate_fft (the reference's algorithm: int64 tonal umbra volumes, scipy
    rfftn/irfftn in f64 with every host thread, rint + projection) on FULL images of the
    config, one image per step (c5: image i of the batch at step i) -- the same config as the
    GPU line.  One c5 call needs ~37 GiB of host RAM and ~16 s on the 16-core box
    (profiles/r2_box_probe.txt)."""
    from oracle import port
    from paper_2305_03018_b200 import workloads as W
    cores = len(os.sched_getaffinity(0))
    if config == "c5":
        se, sd, lo, tmax = W.c5_se(), None, (-15, -15), 63
        image = lambda i: W.c5_image(i % N_IMAGES)  # noqa: E731
    else:
        w = W.CONFIGS[config]()
        se, sd, lo, tmax = w.se_values, w.se_defined, w.se_lo, w.tonal_max
        image = lambda i: w.images[0]  # noqa: E731

    def one(i):
        img = image(i)
        t0 = time.perf_counter()
        if op == "dilate":
            port.dilate_fft(img, None, (0, 0), se, sd, lo, workers=cores)
        else:
            port.erode_fft(img, None, (0, 0), se, sd, lo, l=tmax, workers=cores)
        return time.perf_counter() - t0, img.size

    # bounded: a full c5 image is ~17 s of 16 cores, so a driver-sized run (--steps 20) would
    # take minutes; steps past the time budget are not run (the line says how many were)
    t_start = time.perf_counter()
    for i in range(warmup):
        one(i)
    res = []
    for i in range(steps):
        if res and budget_s is not None:
            mean = sum(t for t, _ in res) / len(res)
            if time.perf_counter() - t_start + mean > budget_s:
                break
        res.append(one(i))
    times = [t for t, _ in res]
    px = sum(n for _, n in res)
    shape = "x".join(str(s) for s in image(0).shape)
    return {"value": px / sum(times) / 1e6, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(times)} full {shape} {config} image(s) (one per step), oracle/port."
                      f"{'dilate_fft' if op == 'dilate' else 'erode_fft'} (reference algorithm: int64 umbra, "
                      f"scipy rfftn/irfftn f64 workers={cores}, rint, project_with_validity)",
            "seconds": sum(times), "steps_s": times}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU algorithm on the box's host cores, same config
    (full images).  A CPU warm-up buys nothing beyond page faults, so at most one warm-up
    step runs (reported as warmup_run)."""
    if rank != 0:
        return
    wu = min(args.warmup, 1)
    budget = float(os.environ.get("FM_REF_BUDGET_S", "150"))
    res = cpu_reference(steps=args.steps, warmup=wu, config=args.config, budget_s=budget)
    ms = 1000.0 * sum(res["steps_s"]) / len(res["steps_s"])
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "warmup_run": wu, "steps_run": len(res["steps_s"]),
        "steps_note": f"one full image per step; steps beyond a {budget:.0f} s host-time budget are not run "
                      "(FM_REF_BUDGET_S)", "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY §8(d) recipe, seeded PCG64)",
        "config": {"workload": WORKLOADS[args.config], "images_per_step": 1, "same_config": True},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _out_digest(values: np.ndarray, valid: np.ndarray) -> str:
    """tests/golden/make_c5_digests.py recipe: sha256(int32 values || uint8 validity)."""
    h = hashlib.sha256(np.ascontiguousarray(values, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(valid, dtype=np.uint8).tobytes())
    return h.hexdigest()


def verify_outputs(out, valid, idx, op):
    """Bit-exact check of every image of a bench batch against the committed reference
    digests (tests/golden/c5_all_digests.json: the C restatement of dilate_naive /
    erode_naive, itself pinned to the reference's own outputs for images 0, 1, 63).
    `out` / `valid` are device or host tensors [n, 2048, 2048]."""
    import torch
    golden = json.loads(GOLDEN.read_text())["images"]
    bad = []

    def one(j):
        i = idx[j]
        v = out[j].to(torch.int32).cpu().numpy()
        m = valid[j].cpu().numpy()
        return i, _out_digest(v, m) == golden[str(i)][op]

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(8) as ex:
        for i, ok in ex.map(one, range(len(idx))):
            if not ok:
                bad.append(i)
    return {"images": len(idx), "ok": not bad, "mismatched": bad}


def over_ranks(value, op, world, device, dtype=None):
    """Reduce one number over the ranks (the bench's only collectives besides the barriers):
    'max' for times (the slowest rank sets the step), 'min' for parity flags, 'sum' for
    counts.  World 1: the value itself."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return value
    t = torch.tensor([value], dtype=dtype or (torch.float64 if isinstance(value, float) else torch.int64),
                     device=device)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op])
    return t.item()


def _timed(fn, steps, stream, world):
    """CUDA-event time of `steps` calls of fn on `stream`, barrier + synchronize on both
    sides, max over ranks (ms)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    return float(over_ranks(float(a.elapsed_time(b)), "max", world,
                            torch.device("cuda", torch.cuda.current_device())))


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2305_03018_b200 import _lib
    from paper_2305_03018_b200 import build as B
    from paper_2305_03018_b200 import workloads as W
    from paper_2305_03018_b200.engine import MorphPlan
    from paper_2305_03018_b200.sharding import shard_range

    B.build_rank_safe(rank, world)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    i0, i1 = shard_range(args.images, rank, world)
    nloc = i1 - i0
    idx = list(range(i0, i1))
    imgs = make_images(idx)
    se = W.c5_se()
    # dilation values of c5 lie in [0, 63 + 15], erosion values in [-15, 63]
    out_dt = {"u8": torch.uint8, "i16": torch.int16, "i32": torch.int32}[args.out_dtype]
    ero_dt = torch.int32 if args.out_dtype == "i32" else torch.int16
    common = dict(shape=(EDGE, EDGE), se_values=se, se_lo=(-15, -15), crop=True, img_dtype=torch.uint8,
                  img_min=0, img_max=63, batch=max(nloc, 1), device=dev, scratch_bytes=args.scratch_gib << 30)
    plan = MorphPlan(mode="dilate", fill=0, out_dtype=out_dt, **common)
    x = torch.from_numpy(imgs).to(dev)
    out = torch.empty((nloc, EDGE, EDGE), dtype=out_dt, device=dev)
    valid = torch.empty((nloc, EDGE, EDGE), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.execute(x, out=out, valid=valid, stream=stream)

    if args.profile_step:
        # exactly one step of the hot path (for an ncu launch list / DRAM-bytes pass)
        step()
        torch.cuda.synchronize()
        print(json.dumps({"profile_step": True, "images": nloc}), flush=True)
        return

    # the clock sampler runs from before the warm-up (all of it under load) to the end
    # of the timed region
    clocks = Clocks(local_rank)
    clocks.wait_first()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.reset_stats()
    torch.cuda.synchronize()
    plan.get_timing(reset=True)
    plan.set_timing(True)
    l0 = _lib.kernel_launches()
    ms = _timed(step, args.steps, stream, world)
    launches = _lib.kernel_launches() - l0
    plan.set_timing(False)
    clk = clocks.stop()
    tim = plan.get_timing(reset=True)
    dev_max = plan.read_stats()
    ms_per_step = ms / args.steps
    mpx = args.images * EDGE * EDGE / 1e6
    value = mpx / (ms_per_step / 1000.0)
    # parity of exactly what was timed: every image of the rank, every pixel
    par_d = verify_outputs(out, valid, idx, "dilate") if args.verify else None

    # e2e: same metric through the public API with HOST buffers (pinned), copies inside.  The
    # host-facing output uses the narrowest type holding every possible value, as the drop-in
    # dilate_fft does (c5: 0..78 -> uint8); --e2e-out-dtype overrides it.
    e2e_dt = {"narrow": torch.uint8, "u8": torch.uint8, "i16": torch.int16, "i32": torch.int32}[args.e2e_out_dtype]
    eplan = plan if e2e_dt == out_dt else MorphPlan(mode="dilate", fill=0, out_dtype=e2e_dt, **common)
    pin_in = torch.from_numpy(imgs).pin_memory()
    pin_out = torch.empty((nloc, EDGE, EDGE), dtype=e2e_dt).pin_memory()
    pin_valid = torch.empty((nloc, EDGE, EDGE), dtype=torch.uint8).pin_memory()
    eplan.execute_host(pin_in, out=pin_out, valid=pin_valid, stream=stream)   # warm (staging alloc)
    e2e_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    e2e_ms = _timed(lambda: eplan.execute_host(pin_in, out=pin_out, valid=pin_valid, stream=stream),
                    e2e_steps, stream, world) / e2e_steps
    wall_ms = (time.perf_counter() - t0) * 1000.0 / e2e_steps
    e2e_val = mpx / (float(over_ranks(float(max(e2e_ms, wall_ms)), "max", world, dev)) / 1000.0)
    par_e2e = verify_outputs(pin_out, pin_valid, idx, "dilate") if args.verify else None
    e2e_osz = pin_out.element_size()
    del pin_in, pin_out, pin_valid
    if eplan is not plan:
        eplan.close()

    # erosion of the same batch (erode_fft semantics, l = tonal_max = 63), same timing rules
    ero = None
    if args.erode:
        eplan = MorphPlan(mode="erode", fill=63, out_dtype=ero_dt, **common)
        eout = torch.empty((nloc, EDGE, EDGE), dtype=ero_dt, device=dev)
        evalid = torch.empty((nloc, EDGE, EDGE), dtype=torch.uint8, device=dev)
        estep = lambda: eplan.execute(x, out=eout, valid=evalid, stream=stream)  # noqa: E731
        for _ in range(max(1, min(args.warmup, 2))):
            estep()
        eplan.reset_stats()
        ems = _timed(estep, args.steps, stream, world) / args.steps
        edev = eplan.read_stats()
        ero = {"value": mpx / (ems / 1000.0), "unit": UNIT, "ms_per_step": ems, "out_dtype": str(ero_dt).split(".")[-1],
               "max_abs_deviation": edev,
               "parity": verify_outputs(eout, evalid, idx, "erode") if args.verify else None}
        del eout, evalid, eplan

    parity = None
    if args.verify:
        flags = [par_d["ok"], par_e2e["ok"]] + ([ero["parity"]["ok"]] if ero else [])
        ok_all = over_ranks(1 if all(flags) else 0, "min", world, dev)
        n_all = over_ranks(nloc, "sum", world, dev)
        parity = {"images": int(n_all), "ok": bool(ok_all),
                  "dilate": par_d, "e2e_dilate": par_e2e, "erode": ero["parity"] if ero else None,
                  "checker": "sha256(int32 values || uint8 validity) per image vs tests/golden/c5_all_digests.json "
                             "(oracle/naive.c restatement of dilate_naive/erode_naive, pinned to the reference "
                             "for images 0, 1, 63)"}

    if rank != 0:
        return
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs")
    peak_note = "measured (MEASURED_PEAKS.json)" if hbm else "fallback (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    conv_s = tim["conv_ms"] / 1000.0 / max(tim["conv_launches"], 1)
    conv_bytes = tim["conv_bytes"] / max(tim["conv_launches"], 1)
    conv_gbs = conv_bytes / conv_s / 1e9 if conv_s > 0 else 0.0
    tonal_s = tim["tonal_ms"] / 1000.0 / max(tim["tonal_launches"], 1)
    tonal_bytes = tim["tonal_bytes"] / max(tim["tonal_launches"], 1)
    sm_mhz = (clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    fp32_peak, fp32_src = _fp32_peak(sm_mhz)
    conv_tflops = tim["conv_flops"] / max(tim["conv_launches"], 1) / conv_s / 1e12 if conv_s > 0 else 0.0
    info = plan.info
    traffic, traffic_src, pipe, dram_step = _ncu_traffic(info["images_per_launch"], args.images)
    fpp = 2.0 * 5.0 * 128 * 128 * math.log2(128 * 128) + 6.0 * 128 * 128
    tiles = info["tiles_y"] * info["tiles_x"]
    mean_planes = tim["conv_flops"] / fpp / (tiles * args.images * args.steps) if tim["conv_flops"] else None
    osz = torch.empty((), dtype=out_dt).element_size()
    fft_bytes = tim["conv_bytes"] + tim["tonal_bytes"]
    fft_s = (tim["conv_ms"] + tim["tonal_ms"]) / 1000.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "dtype_note": "FFT arithmetic in FP32 (the reference uses f64); spectral planes between the passes stored "
                      "as int16 pairs at a per-tile fixed-point scale (analytic count error <= sqrt(2) C/64000, "
                      f"C = defined SE entries); exact integer results: worst pre-rounding deviation {dev_max:.2e}, "
                      f"margin {0.5 / max(dev_max, 1e-30):.0f}x to 0.5",
        "data": "synthetic (SURVEY §8(d) c5 recipe, seeded PCG64)",
        "config": {"workload": WORKLOAD, "images": args.images, "images_per_gpu": nloc,
                   "out_dtype": args.out_dtype, "tonal_len": info["tonal_len"],
                   "planes_max": info["planes"], "mean_planes_per_tile": mean_planes,
                   "tile": [info["tile_y"], info["tile_x"]], "tiles_per_image": tiles,
                   "window": [info["valid_y"], info["valid_x"]],
                   "images_per_launch": info["images_per_launch"],
                   "l2": "no flush: inputs 256 MiB and the spectral volume (~0.7 GB/image at "
                         f"{(mean_planes or 0):.1f} planes/tile) exceed the 126 MB L2"},
        # the dominant kernel (conv, ~80% of the step) is bound by the FP32 pipe, not HBM
        "roofline": {"bound": "fp32", "kernel": "tile128_kernel (encode + three-pass 2-D FFT conv, fm_tile128.cuh)",
                     "achieved": conv_tflops, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": conv_tflops / fp32_peak if fp32_peak else None,
                     "peak_source": fp32_src,
                     "flops_note": "nominal 2*5*P^2*log2(P^2)+6*P^2 per (tile, plane), P=128, summed over the "
                                   "planes actually computed",
                     "traffic": traffic, "traffic_source": traffic_src,
                     "ms_per_launch": conv_s * 1000.0, "ncu_pct": pipe,
                     "hbm_view": {"achieved": conv_gbs, "peak": hbm, "unit": "GB/s", "frac": conv_gbs / hbm,
                                  "bytes_per_launch": conv_bytes, "peak_source": peak_note},
                     "tonal_kernel": {"achieved": tonal_bytes / tonal_s / 1e9 if tonal_s > 0 else 0.0,
                                      "unit": "GB/s", "frac": (tonal_bytes / tonal_s / 1e9) / hbm if tonal_s > 0 else 0.0,
                                      "ms_per_launch": tonal_s * 1000.0},
                     # SURVEY §8(d) graded figure: sum of the FFT passes' logical bytes over their summed time
                     "fft_passes": {"bytes_per_step": fft_bytes / args.steps, "achieved": fft_bytes / fft_s / 1e9 if fft_s else 0.0,
                                    "unit": "GB/s", "frac": fft_bytes / fft_s / 1e9 / hbm if fft_s else 0.0},
                     # the range kernels run one launch chunk ahead on a low-priority stream
                     # (overlapping the conv tail / tonal kernels): their event span is not a
                     # share of the step
                     "share_of_step": {"conv": tim["conv_ms"] / max(ms, 1e-9), "tonal": tim["tonal_ms"] / max(ms, 1e-9)},
                     "dram_bytes_per_step": dram_step,
                     # the whole path against the method's HBM floor: EFFECTIVE -- the per-tile
                     # tonal length moves less than the floor's minimal-extent volume
                     "method_floor_effective": method_floor(value, hbm, osz)},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(imgs.nbytes),
                "d2h_bytes_per_step": int(nloc * EDGE * EDGE * (e2e_osz + 1)),
                "out_dtype": str(e2e_dt).split(".")[-1], "api": "fm_execute_host (pinned host buffers)"},
        "gpu_launches": int(launches),
        "max_abs_deviation": dev_max,
        "parity": parity,
        "erode": ero,
        "clocks": clk,
    }
    if args.cpu_baseline and world == 1:
        try:
            cb = cpu_reference(steps=1)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # keep the GPU line even if the host baseline fails (e.g. RAM)
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                                    "kind": "port", "sample": f"failed: {type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)
    if args.verify and not parity["ok"]:
        sys.exit(3)


def run_strips(args, rank, world, local_rank):
    """--config c3|c4: ONE image per step, split into row strips across the ranks (one process
    per GPU, sharding.strips geometry); halo rows by NVLink peer copies out of the neighbours'
    IPC-mapped strip buffers inside the timed region (strips.RankStrip); each rank computes
    exactly its owned output rows.  N = 1: the whole image on one GPU."""
    import torch
    import torch.distributed as dist
    from paper_2305_03018_b200 import _lib
    from paper_2305_03018_b200 import build as B
    from paper_2305_03018_b200 import workloads as W
    from paper_2305_03018_b200.engine import MorphPlan
    from paper_2305_03018_b200.strips import RankStrip

    B.build_rank_safe(rank, world)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = W.CONFIGS[args.config]()
    img = w.images[0]
    H, Wd = img.shape
    sd = None if w.se_defined.all() else w.se_defined
    stream = torch.cuda.current_stream(dev)
    kw = dict(se_values=w.se_values, se_lo=w.se_lo, se_defined=sd, mode="dilate", img_dtype=torch.uint8,
              img_min=0, img_max=w.tonal_max, fill=0, out_dtype=torch.int32, device=dev)
    if world > 1:
        rs = RankStrip(rank=rank, world=world, shape=img.shape, **kw)
        me = rs.me
        rs.load_own(torch.from_numpy(img[me.out0:me.out1]).to(dev))
        out = torch.empty((1, me.out1 - me.out0, Wd), dtype=torch.int32, device=dev)
        valid = torch.empty_like(out, dtype=torch.uint8)
        torch.cuda.synchronize()
        dist.barrier()

        def step():
            rs.exchange_halos(stream)
            rs.execute(stream, out=out, valid=valid)
        plan, rows = rs.plan, (me.out0, me.out1)
    else:
        plan = MorphPlan(shape=img.shape, crop=True, batch=1, **kw)
        x = torch.from_numpy(img).to(dev).unsqueeze(0)
        out = torch.empty((1, H, Wd), dtype=torch.int32, device=dev)
        valid = torch.empty_like(out, dtype=torch.uint8)

        def step():
            plan.execute(x, out=out, valid=valid, stream=stream)
        rows = (0, H)
    clocks = Clocks(local_rank)
    clocks.wait_first()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    plan.reset_stats()
    l0 = _lib.kernel_launches()
    ms = _timed(step, args.steps, stream, world)
    launches = _lib.kernel_launches() - l0
    clk = clocks.stop()
    dev_max = plan.read_stats()
    ms_per_step = ms / args.steps
    mpx = H * Wd / 1e6
    value = mpx / (ms_per_step / 1000.0)
    # e2e: this rank's own input rows H2D from pinned memory and its output rows D2H, inside
    # the timed region (plus the halo copies and compute)
    r0, r1 = rows
    pin_in = torch.from_numpy(img[r0:r1]).pin_memory()
    pin_out = torch.empty((r1 - r0, Wd), dtype=torch.int32).pin_memory()
    pin_valid = torch.empty((r1 - r0, Wd), dtype=torch.uint8).pin_memory()

    def e2e_step():
        if world > 1:
            rs.window[me.out0 - me.in0: me.out1 - me.in0].copy_(pin_in, non_blocking=True)
            stream.synchronize()
            dist.barrier()     # neighbours' rows landed before the halo copies read them
            step()
        else:
            x[0].copy_(pin_in, non_blocking=True)
            step()
        pin_out.copy_(out[0], non_blocking=True)
        pin_valid.copy_(valid[0], non_blocking=True)
        stream.synchronize()
    e2e_step()
    t0 = time.perf_counter()
    e2e_ms = _timed(e2e_step, args.steps, stream, world) / args.steps
    wall_ms = (time.perf_counter() - t0) * 1000.0 / args.steps
    e2e_val = mpx / (float(over_ranks(float(max(e2e_ms, wall_ms)), "max", world, dev)) / 1000.0)
    # parity: the stitched image against the reference's own output digest
    parts = [None] * world
    mine = (r0, pin_out.numpy().copy(), pin_valid.numpy().copy())
    if world > 1:
        dist.all_gather_object(parts, mine)
    else:
        parts = [mine]
    parity = None
    if rank == 0:
        parts.sort(key=lambda t: t[0])
        vals = np.concatenate([p[1] for p in parts])
        vm = np.concatenate([p[2] for p in parts])
        golden = json.loads((ROOT / "tests" / "golden" / "digests.json").read_text())[f"{args.config}_img0"]
        parity = {"images": 1, "ok": _out_digest(vals, vm) == golden["dilate"],
                  "checker": "sha256(int32 values || uint8 validity) of the stitched strips vs the reference's "
                             "dilate_naive output (tests/golden/digests.json)"}
    if world > 1:
        rs.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SURVEY §8(d) recipe, seeded PCG64)",
        "config": {"workload": WORKLOADS[args.config], "strips": world, "tonal_len": plan.info["tonal_len"],
                   "tile": [plan.info["tile_y"], plan.info["tile_x"]],
                   "l2": "no flush: single image per step; the spectral scratch exceeds L2"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(img.nbytes),
                "d2h_bytes_per_step": int(H * Wd * 5)},
        "gpu_launches": int(launches), "max_abs_deviation": dev_max, "parity": parity, "clocks": clk,
    }
    if args.cpu_baseline and world == 1:
        try:
            cb = cpu_reference(steps=1, config=args.config)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                                    "kind": "port", "sample": f"failed: {type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)
    if parity is not None and not parity["ok"]:
        sys.exit(3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c5", "c3", "c4"], default="c5",
                    help="c5: the 64-image batch sharded by image (headline); c3/c4: one image in row strips")
    ap.add_argument("--images", type=int, default=N_IMAGES)
    ap.add_argument("--scratch-gib", type=int, default=16)
    ap.add_argument("--out-dtype", choices=["u8", "i16", "i32"], default="i32",
                    help="output value type (int32 as SURVEY §8(d); the c5 dilation range 0..78 also fits u8)")
    ap.add_argument("--e2e-out-dtype", choices=["narrow", "u8", "i16", "i32"], default="narrow",
                    help="host output type of the e2e run (narrow: the narrowest type holding every value, "
                         "as the drop-in API picks)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-verify", dest="verify", action="store_false",
                    help="skip the post-timing bit-exact check of every output image")
    ap.add_argument("--no-erode", dest="erode", action="store_false", help="skip the erosion measurement")
    ap.add_argument("--profile-step", action="store_true",
                    help="run exactly one untimed step and exit (for profilers)")
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
        if args.config == "c5":
            run_ours(args, rank, world, local_rank)
        else:
            run_strips(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
