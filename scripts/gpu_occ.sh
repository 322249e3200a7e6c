#!/bin/bash
mkdir -p gpurun_out
for o in 64 4 3; do FM_TONAL_OCC=$o timeout 600 python scripts/bench_configs.py --only c5 > gpurun_out/configs_occ$o.log 2>&1; done
