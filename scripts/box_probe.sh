#!/bin/bash
# Host facts of the GPU box + one full-size (2048^2) c5 reference-algorithm call (oracle/port).
mkdir -p gpurun_out
{
  nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"
  nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
  python - <<'PY'
import os, time, resource, sys
sys.path.insert(0, ".")
from oracle import port
from paper_2305_03018_b200 import workloads as W
img = W.c5_image(0); se = W.c5_se()
cores = len(os.sched_getaffinity(0))
t = time.perf_counter()

r = port.dilate_fft(img, None, (0, 0), se, None, (-15, -15), workers=cores)
print("full 2048^2 dilate_fft s", time.perf_counter() - t, "cores", cores,
      "maxrss GiB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20, flush=True)
PY
} > gpurun_out/box_probe.txt 2>&1
