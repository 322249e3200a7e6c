#!/bin/bash
# usage: bash scripts/gpu_ncu_conv.sh TAG [REGEX] — ncu --set full of one conv launch (4-image c5 bench)
TAG=${1:-run}; RX=${2:-tile128_kernelIhLb0E}
mkdir -p gpurun_out
timeout 300 python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$RX" -s 1 -c 1 -o gpurun_out/prof_$TAG \
   python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_$TAG.log
