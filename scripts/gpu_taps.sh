#!/bin/bash
mkdir -p gpurun_out
for t in 128 64 32 16; do
  FM_RANGE_TAPS=$t timeout 600 python scripts/bench_configs.py --modes dilate > gpurun_out/configs_taps$t.log 2>&1
done
